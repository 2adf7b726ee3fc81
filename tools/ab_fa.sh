python -m paper_2411_02820_b200._build > /dev/null 2>&1
mkdir -p gpurun_out/ab1
for e in 0 1 2 3 0; do echo "EMU=$e"; DS_FA_EMU=$e timeout 120 python tools/attn_bench.py; done > gpurun_out/ab1/attn.log 2>&1
DS_FA_EMU=2 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k attention > gpurun_out/ab1/tests2.log 2>&1
DS_FA_EMU=3 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k attention > gpurun_out/ab1/tests3.log 2>&1
