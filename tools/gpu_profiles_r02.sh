#!/bin/bash
# Round-2 evidence: GPU suite, smoke, full bench (with the CPU leg), fan-out code path (batched) on one GPU,
# launch list of one consumer step, full ncu captures (step kernels, batched anchor kernels).
#   gpurun --timeout 3600 -- bash tools/gpu_profiles_r02.sh <tag>
OUT=gpurun_out/${1:-r02_final}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --steps 5 --warmup 3 --same-device --batch 4 > $OUT/fanout_same_device_b4.log 2>&1; echo "rc=$?" >> $OUT/fanout_same_device_b4.log
bash tools/prof_step.sh ${1:-r02_final}/step > /dev/null 2>&1
NCU="ncu --profile-from-start off --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:"gemv_batch|attn_batch" -c 5 -o $OUT/prof_batch python tools/anchor_alone.py --batch 4 --profile > $OUT/ncu_batch.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
    --log-file $OUT/launches_anchor_b4.csv python tools/anchor_alone.py --batch 4 --profile > /dev/null 2>&1
ls -la $OUT $OUT/step
# keep the copy-back under 64 MiB: raw-page CSVs of every capture, drop the big reports
for r in $(find $OUT -name "*.ncu-rep"); do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
done
find $OUT -name "*.ncu-rep" -size +8M -delete
du -sh $OUT
