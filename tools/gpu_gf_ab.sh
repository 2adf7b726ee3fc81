#!/bin/bash
OUT=gpurun_out/${1:-gf_ab}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for r in 0 1; do for b in 0 8; do
  echo "head b=$b $(DS_LIB=ab/att_head.so timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-90)"
  echo "new  b=$b $(timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-90)"
done; done > $OUT/ab.txt 2>&1
for r in 0 1 2; do
  echo "head $(DS_LIB=ab/att_head.so timeout 300 python tools/step_time.py 2>&1 | tail -1)"
  echo "new  $(timeout 300 python tools/step_time.py 2>&1 | tail -1)"
done >> $OUT/ab.txt 2>&1
cat $OUT/ab.txt
