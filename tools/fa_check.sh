set -x
OUT=gpurun_out/fa1; mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > $OUT/attn_tests.log 2>&1
timeout 120 python tools/attn_bench.py > $OUT/attn_new.log 2>&1
DS_FA_LEGACY=1 timeout 120 python tools/attn_bench.py > $OUT/attn_legacy.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --full-steps 3 > $OUT/bench.log 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_partial.csv python tools/profile_step.py --what partial > $OUT/ncu_launch.log 2>&1
