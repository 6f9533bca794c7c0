#!/bin/bash
# A/B helper over library builds: alternate bench runs (no CPU baseline) with each listed
# _lib/<variant> (or "main") on one box.  usage: tools/ab_libs.sh rounds variant...
N="$1"; shift
mkdir -p gpurun_out
for i in $(seq 1 "$N"); do
  for v in "$@"; do
    if [ "$v" = main ]; then lib=""; else lib="$PWD/paper_2101_06354_b200/_lib/$v/libssimk.so"; fi
    SSK_LIBRARY="$lib" python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/ab.json 2>/dev/null
    python - "$v" <<'PY'
import json, sys; d = json.load(open("gpurun_out/ab.json"))
print(f"{sys.argv[1]:8s} value {d['value']:9.0f}  ms_step {d['ms_per_step']:.4f}  k_ms {d['roofline']['kernel_ms']:.4f}")
PY
  done
done
