#!/bin/bash
OUT=gpurun_out/${1:-batch3}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_batch.py tests/test_gpu_shapes.py -q -x > $OUT/pytest_batch.log 2>&1; echo "rc=$?" >> $OUT/pytest_batch.log
tail -2 $OUT/pytest_batch.log
for b in 0 2 4 8; do timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-110; done > $OUT/times.txt
cat $OUT/times.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --steps 5 --warmup 3 --same-device --batch 4 > $OUT/fanout_b4.log 2>&1; echo "rc=$?" >> $OUT/fanout_b4.log
grep -o '"ttft_p50_ms": [0-9.]*' $OUT/fanout_b4.log | head -1; tail -2 $OUT/fanout_b4.log | cut -c1-300
