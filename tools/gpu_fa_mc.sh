#!/bin/bash
OUT=gpurun_out/${1:-fa_mc}
mkdir -p $OUT
DS_FA_VARIANT=5 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for r in 0 1; do for v in 3 5; do echo "v$v $(DS_FA_VARIANT=$v timeout 120 python tools/attn_bench.py 2>&1 | tail -1)"; done; done > $OUT/ab.txt 2>&1
echo "abl v5 $(DS_FA_VARIANT=5 DS_LIB=ab/fa_abl1.so timeout 120 python tools/attn_bench.py 2>&1 | tail -1)" >> $OUT/ab.txt
DS_FA_VARIANT=5 DS_LIB=ab/fa_stamps.so timeout 120 python tools/attn_bench.py > $OUT/stamps.txt 2>&1
cat $OUT/ab.txt; sed -n 8,14p $OUT/stamps.txt
for r in 0 1 2; do for v in 3 5; do echo "v$v $(DS_FA_VARIANT=$v timeout 300 python tools/step_time.py 2>&1 | tail -1)"; done; done > $OUT/step.txt 2>&1
cat $OUT/step.txt
