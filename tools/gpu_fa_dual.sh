#!/bin/bash
OUT=gpurun_out/${1:-fa_dual}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > $OUT/pytest_att.log 2>&1; echo "rc=$?" >> $OUT/pytest_att.log
tail -3 $OUT/pytest_att.log
for r in 0 1; do for v in 1 3; do echo "variant=$v $(DS_FA_VARIANT=$v timeout 120 python tools/attn_bench.py 2>&1 | tail -1)"; done; done > $OUT/variants.txt 2>&1
cat $OUT/variants.txt
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --batch-leg "" > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
grep -o '"ttft_p50_ms": [0-9.]*' $OUT/bench.log | head -2; grep -o '"attention_prefill": {[^}]*}' $OUT/bench.log
