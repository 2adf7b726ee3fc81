#!/bin/bash
# ncu full captures of the FA prefill kernel and the recompute GEMMs (one consumer step)
OUT=gpurun_out/${1:-prof2}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 400 python -m pytest tests/test_gpu_quality.py tests/test_gpu_parity.py -q -x > $OUT/pytest.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fa_tc -s 3 -c 1 -o $OUT/fa python tools/attn_bench.py > $OUT/ncu_fa.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tcgen05 -c 5 -o $OUT/gemm python tools/profile_step.py --what partial > $OUT/ncu_gemm.log 2>&1
timeout 300 python tools/overlap_probe.py > $OUT/probe.json 2> $OUT/probe.err
