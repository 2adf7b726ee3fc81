#!/bin/bash
OUT=gpurun_out/${1:-fa_one}
mkdir -p $OUT
DS_FA_VARIANT=4 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for r in 0 1; do for v in 3 4; do echo "v$v $(DS_FA_VARIANT=$v timeout 120 python tools/attn_bench.py 2>&1 | tail -1)"; done; done > $OUT/ab.txt 2>&1
cat $OUT/ab.txt
for r in 0 1 2; do for v in 3 4; do echo "v$v $(DS_FA_VARIANT=$v timeout 300 python tools/step_time.py 2>&1 | tail -1)"; done; done > $OUT/step.txt 2>&1
cat $OUT/step.txt
