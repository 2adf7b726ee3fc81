#!/bin/bash
OUT=gpurun_out/${1:-att_ab2}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_batch.py tests/test_gpu_8b.py tests/test_gpu_parity.py tests/test_gpu_8b_numerics.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for r in 0 1; do for b in 0 8; do
  echo "head b=$b $(DS_LIB=ab/att_head.so timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-90)"
  echo "new  b=$b $(timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-90)"
done; done > $OUT/ab.txt 2>&1
for r in 0 1 2; do for L in att_head new; do
  if [ $L = new ]; then echo "new  $(timeout 300 python tools/step_time.py 2>&1 | tail -1)"; else echo "head $(DS_LIB=ab/att_head.so timeout 300 python tools/step_time.py 2>&1 | tail -1)"; fi
done; done >> $OUT/ab.txt 2>&1
cat $OUT/ab.txt
