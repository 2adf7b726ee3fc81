#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench, ncu launch list (+ full capture unless quick).
#   gpurun --timeout 2400 -- bash tools/gpu_check.sh <tag> [quick|full] [kernel-regex]
set -x
TAG=${1:-r01}
MODE=${2:-full}
KREGEX=${3:-"gemm_tcgen05|fa_prefill|kv_ingest|gemv|decode_attn"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
if [ "$MODE" = quick ]; then
  timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
else
  timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
fi
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_partial.csv python tools/profile_step.py --what partial > $OUT/ncu_launch.log 2>&1
if [ "$MODE" != quick ]; then
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"$KREGEX" -c 14 -o $OUT/prof_partial python tools/profile_step.py --what partial > $OUT/ncu_full.log 2>&1
fi
ls -la $OUT
