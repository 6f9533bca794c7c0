#!/bin/bash
# A/B of the end-to-end rate under two environment settings, interleaved on one box.
# usage: tools/ab_e2e.sh "VAR=a ..." "VAR=b ..." [rounds]
A="$1"; B="$2"; N="${3:-3}"
for i in $(seq 1 "$N"); do
  for e in "$A" "$B"; do
    env $e python bench.py --steps 40 --warmup 5 --no-cpu 2>/dev/null | python -c "
import json, sys; d = json.load(sys.stdin)
print(f'{sys.argv[1]:40s} value {d[\"value\"]:9.0f}  e2e {d[\"e2e\"][\"value\"]:8.0f}  e2e ms {d[\"e2e\"][\"ms_per_step\"]:.3f}')" "$e"
  done
done
