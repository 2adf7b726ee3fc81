#!/bin/bash
# Anchor-shape crossover: the config-5 points with the persistent co-resident
# anchor forced and with the per-launch anchor forced (compare the two JSONs).
#   gpurun --timeout 2400 -- bash tools/crossover.sh <tag>
OUT=gpurun_out/${1:-xover}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
for shape in persistent launch; do
  DS_ANCHOR_SHAPE=$shape timeout 900 python tools/sweep.py --ns 2048,4096,8192,16384 --ks 3,6,10,16 --steps 5 \
      > $OUT/sweep_$shape.json 2>> $OUT/sweep.err
done
ls -la $OUT
