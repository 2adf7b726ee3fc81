#!/bin/bash
# Second rows of config 2 (SwiGLU MLP) and config 3's Mistral-7B shape (V=32000), one GPU.
OUT=gpurun_out/${1:-rows}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_swiglu.py tests/test_gpu_kernels.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py --mlp swiglu --no-cpu-baseline > $OUT/bench_swiglu.log 2>&1; echo "rc=$?" >> $OUT/bench_swiglu.log
timeout 900 python bench.py --vocab 32000 --no-cpu-baseline > $OUT/bench_mistral.log 2>&1; echo "rc=$?" >> $OUT/bench_mistral.log
