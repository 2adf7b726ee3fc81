#!/bin/bash
OUT=gpurun_out/${1:-att_ncu}
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_decode_tma_kernel" -s 40 -c 1 -o $OUT/att python tools/anchor_alone.py --reps 1 > $OUT/ncu.log 2>&1
ncu -i $OUT/att.ncu-rep --page source --csv > $OUT/att_source.csv 2>&1
ncu -i $OUT/att.ncu-rep --page raw --csv > $OUT/att_raw.csv 2>&1
ls -la $OUT
