python -m paper_2411_02820_b200._build > /dev/null 2>&1
mkdir -p gpurun_out/ab4
for g in 16 64 8; do echo "GROUP=$g"; DS_GEMM_GROUP=$g timeout 120 python tools/gemm_bench.py; DS_GEMM_GROUP=$g timeout 300 python tools/overlap_probe.py; done > gpurun_out/ab4/group.log 2>&1
