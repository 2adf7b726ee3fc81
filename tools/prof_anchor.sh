#!/bin/bash
# Stand-alone anchor pass (ds_anchor, per-launch kernels): timing, launch list
# (warm L2: --cache-control none) and full captures of one layer's kernels.
#   gpurun --timeout 1500 -- bash tools/prof_anchor.sh <tag>
OUT=gpurun_out/${1:-anchor}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 300 python tools/anchor_alone.py > $OUT/time.json 2> $OUT/time.err
timeout 300 python tools/anchor_alone.py --n 2048 > $OUT/time_2k.json 2>> $OUT/time.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none \
    --cache-control none --csv --log-file $OUT/launches.csv python tools/anchor_alone.py --profile > $OUT/ncu_launch.log 2>&1
if [ -n "$FULL" ]; then
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"gemv|attn_decode" -c 5 -o $OUT/prof python tools/anchor_alone.py --profile > $OUT/ncu_full.log 2>&1
fi
ls -la $OUT
cat $OUT/time.json $OUT/time_2k.json
