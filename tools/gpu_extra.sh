#!/bin/bash
# Extra GPU checks: quality/IPC tests, sweep, fan-out bench on one GPU (2 ranks, same device).
set -x
OUT=gpurun_out/${1:-extra}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_quality.py tests/test_gpu_ipc.py -x -q -s > $OUT/pytest_quality.log 2>&1; echo "rc=$?" >> $OUT/pytest_quality.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --same-device > $OUT/fanout_same_device.log 2>&1; echo "rc=$?" >> $OUT/fanout_same_device.log
timeout 900 python tools/sweep.py --steps 5 > $OUT/sweep.json 2> $OUT/sweep.log; echo "rc=$?" >> $OUT/sweep.log
