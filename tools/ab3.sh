python -m paper_2411_02820_b200._build > /dev/null 2>&1
mkdir -p gpurun_out/ab3
timeout 120 python tools/gemm_bench.py > gpurun_out/ab3/gemm.log 2>&1
timeout 120 python tools/attn_bench.py > gpurun_out/ab3/attn.log 2>&1
timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/ab3/pytest.log 2>&1
timeout 300 python tools/overlap_probe.py > gpurun_out/ab3/probe.json 2>&1
