#!/bin/bash
# GPU suite + stand-alone / batched anchor times.
OUT=gpurun_out/${1:-check_anchor}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
for b in 0 2 4 8; do timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-110; done > $OUT/times.txt
cat $OUT/times.txt
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file $OUT/launch_b4.csv python tools/anchor_alone.py --batch 4 --profile > /dev/null 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file $OUT/launch_b0.csv python tools/anchor_alone.py --profile > /dev/null 2>&1
