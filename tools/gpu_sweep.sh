#!/bin/bash
# GPU tests, then the config-5 sweep (n x k) into gpurun_out/<tag>/sweep.json
OUT=gpurun_out/${1:-sweep}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -2 $OUT/pytest_gpu.log
timeout 1500 python tools/sweep.py > $OUT/sweep.json 2> $OUT/sweep.err; tail -2 $OUT/sweep.err
