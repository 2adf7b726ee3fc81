#!/bin/bash
# Claimed GEMV tiles (GemvArgs::tile_ctr) vs blockIdx-strided (DS_GEMV_CLAIM=0): GPU suite, then
# same-box A/B of the stand-alone anchor chain and of the consumer step.
OUT=gpurun_out/${1:-claim}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log
for r in 0 1 2; do for c in 0 1; do
  echo "claim=$c $(DS_GEMV_CLAIM=$c timeout 300 python tools/anchor_alone.py --reps 10 2>&1 | tail -1 | cut -c1-90)"
done; done > $OUT/ab.txt 2>&1
for r in 0 1; do for c in 0 1; do
  echo "claim=$c $(DS_GEMV_CLAIM=$c timeout 300 python tools/step_time.py 2>&1 | tail -1)"
done; done >> $OUT/ab.txt 2>&1
cat $OUT/ab.txt
