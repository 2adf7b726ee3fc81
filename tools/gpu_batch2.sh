#!/bin/bash
# Batch path after the 2-rows-per-warpgroup GEMV + pinned roundings; FA stamps/ablation; full suite; bench.
OUT=gpurun_out/${1:-batch2}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_batch.py -q > $OUT/pytest_batch.log 2>&1; echo "rc=$?" >> $OUT/pytest_batch.log
tail -4 $OUT/pytest_batch.log
timeout 300 python tools/batch_debug.py > $OUT/batch_debug.txt 2>&1; grep -c diffs $OUT/batch_debug.txt
DS_LIB=ab/fa_stamps.so timeout 120 python tools/attn_bench.py > $OUT/fa_stamps.txt 2>&1
for r in 0 1; do for v in main fa_abl1; do
  if [ $v = main ]; then echo "main $(timeout 120 python tools/attn_bench.py 2>&1 | tail -1)";
  else echo "$v $(DS_LIB=ab/$v.so timeout 120 python tools/attn_bench.py 2>&1 | tail -1)"; fi
done; done > $OUT/fa_ab.txt 2>&1; cat $OUT/fa_ab.txt
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
grep -o '"batch": {.*"n_tokens"' $OUT/bench.log | head -c 1200; echo; grep -o '"ttft_p50_ms": [0-9.]*' $OUT/bench.log | head -2
