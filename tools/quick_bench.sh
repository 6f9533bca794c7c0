#!/bin/bash
# quick A/B helper: two short bench runs (no CPU baseline) + the GPU test suite
mkdir -p gpurun_out
for i in 1 2; do
python bench.py --no-cpu --steps 30 > gpurun_out/qb_$i.json 2>/dev/null
python - "$i" <<'PY'
import json, sys; d=json.load(open(f"gpurun_out/qb_{sys.argv[1]}.json"))
print("value", round(d["value"]), "ms_step", round(d["ms_per_step"],4), "k_ms", round(d["roofline"]["kernel_ms"],4), "frac", round(d["roofline"]["frac"],4), "e2e", round(d["e2e"]["value"]))
PY
done
if [ "$1" != "notest" ]; then python -m pytest tests -m gpu -x -q 2>&1 | tail -2; fi
