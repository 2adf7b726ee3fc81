#!/bin/bash
OUT=gpurun_out/${1:-fa_ab2}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for r in 0 1; do for v in 0 1 2; do echo "variant=$v $(DS_FA_VARIANT=$v timeout 120 python tools/attn_bench.py 2>&1 | tail -1)"; done; done > $OUT/variants.txt
