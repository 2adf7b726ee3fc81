#!/bin/bash
# Batched-request path: build, batch tests, full GPU suite, bench with the config-4 leg.
#   gpurun --timeout 2400 -- bash tools/gpu_batch.sh <tag>
OUT=gpurun_out/${1:-batch}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > $OUT/pytest_batch.log 2>&1; echo "rc=$?" >> $OUT/pytest_batch.log
tail -15 $OUT/pytest_batch.log
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -5 $OUT/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
tail -c 1500 $OUT/bench.log
