#!/bin/bash
# Batched GEMV layout A/B (rows per warpgroup) on one box.
OUT=gpurun_out/${1:-gemvb_ab}
mkdir -p $OUT
for lib in main gb_nbw1 gb_nbw4; do
  if [ $lib = main ]; then L=""; else L="ab/$lib.so"; fi
  for b in 2 4; do echo "$lib b=$b $(DS_LIB=$L timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-110)"; done
  DS_LIB=$L timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file $OUT/launch_$lib.csv python tools/anchor_alone.py --batch 4 --profile > /dev/null 2>&1
done > $OUT/times.txt 2>&1
cat $OUT/times.txt
