#!/bin/bash
# FA iteration: attention tests, stamps, stand-alone and in-step A/B against ab/fa_head.so.
OUT=gpurun_out/${1:-fa_iter}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
DS_LIB=ab/fa_stamps.so timeout 120 python tools/attn_bench.py > $OUT/stamps.txt 2>&1; sed -n 10,14p $OUT/stamps.txt
for r in 0 1; do
  echo "head $(DS_LIB=ab/fa_head.so timeout 120 python tools/attn_bench.py 2>&1 | tail -1)"
  echo "new  $(timeout 120 python tools/attn_bench.py 2>&1 | tail -1)"
done > $OUT/ab.txt 2>&1
for r in 0 1 2; do
  echo "head $(DS_LIB=ab/fa_head.so timeout 300 python tools/step_time.py 2>&1 | tail -1)"
  echo "new  $(timeout 300 python tools/step_time.py 2>&1 | tail -1)"
done >> $OUT/ab.txt 2>&1
cat $OUT/ab.txt
