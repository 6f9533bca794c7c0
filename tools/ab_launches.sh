#!/bin/bash
# Per-kernel times (ncu launch list: cold-cache, serialised) of one MS-SSIM step and of the
# score-only level-0 launch, for each listed library variant (_lib/<variant>, or "main").
# usage: tools/ab_launches.sh variant...
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = main ]; then lib=""; else lib="$PWD/paper_2101_06354_b200/_lib/$v/libssimk.so"; fi
  for mode in step l0; do
    SSK_LIBRARY="$lib" ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${v}_${mode}.csv python tools/prof_driver.py --mode $mode --reps 3 > /dev/null 2>&1
    echo "== $v $mode"
    python tools/launch_shares.py gpurun_out/launches_${v}_${mode}.csv
  done
done
