#!/bin/bash
# ncu --set full of one prefill-attention launch (source-level stalls).
OUT=gpurun_out/${1:-fa_ncu}; mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fa_tc" -s 3 -c 1 -o $OUT/fa python tools/attn_bench.py > $OUT/ncu.log 2>&1
ncu -i $OUT/fa.ncu-rep --page source --csv > $OUT/fa_source.csv 2>&1
ncu -i $OUT/fa.ncu-rep --page raw --csv > $OUT/fa_raw.csv 2>&1
ls -la $OUT
