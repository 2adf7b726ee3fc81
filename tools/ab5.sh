python -m paper_2411_02820_b200._build > /dev/null 2>&1
mkdir -p gpurun_out/ab5
timeout 120 python tools/attn_bench.py > gpurun_out/ab5/attn.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > gpurun_out/ab5/tests.log 2>&1
