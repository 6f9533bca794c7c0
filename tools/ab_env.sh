#!/bin/bash
# A/B helper: alternate bench runs (no CPU baseline) under two environment settings on one box.
# usage: tools/ab_env.sh "VAR=a" "VAR=b" [rounds]
A="$1"; B="$2"; N="${3:-3}"
mkdir -p gpurun_out
for i in $(seq 1 "$N"); do
  for e in "$A" "$B"; do
    env $e python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/ab.json 2>/dev/null
    python - "$e" <<'PY'
import json, sys; d = json.load(open("gpurun_out/ab.json"))
print(f"{sys.argv[1]:28s} value {d['value']:9.0f}  ms_step {d['ms_per_step']:.4f}  k_ms {d['roofline']['kernel_ms']:.4f}")
PY
  done
done
