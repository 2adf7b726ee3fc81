#!/bin/bash
# Round check: all GPU tests, smoke, bench (N=1), fan-out code path on one GPU, launch list.
#   gpurun --timeout 2400 -- bash tools/gpu_round.sh <tag>
OUT=gpurun_out/${1:-round}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --steps 5 --warmup 3 --same-device --batch 2 > $OUT/fanout_same_device.log 2>&1; echo "rc=$?" >> $OUT/fanout_same_device.log
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_partial.csv python tools/profile_step.py --what partial > $OUT/ncu_launch.log 2>&1
