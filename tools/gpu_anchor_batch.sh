#!/bin/bash
# Batched anchor pass: event times for 1/2/4/8 rows; ncu launch lists for 1 and 4 rows.
OUT=gpurun_out/${1:-anchor_batch}
mkdir -p $OUT
for b in 0 2 4 8; do timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-200; done > $OUT/times.txt
cat $OUT/times.txt
for b in 0 4; do
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none \
  --csv --log-file $OUT/launch_b$b.csv python tools/anchor_alone.py --batch $b --profile > /dev/null 2>&1
done
ls $OUT
