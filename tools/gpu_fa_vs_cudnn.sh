#!/bin/bash
# ncu --set full of one prefill-attention launch each: ours (fa_dual_kernel, the
# default) and cuDNN's sm100 SDPA at the 8B shape; then both timed on the box.
OUT=gpurun_out/${1:-fa_vs_cudnn}; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fa_dual" -s 3 -c 1 -o $OUT/ours python tools/attn_bench.py > $OUT/ncu_ours.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"sdpa|fmha|flash" -s 2 -c 1 -o $OUT/cudnn python tools/attn_cudnn_once.py > $OUT/ncu_cudnn.log 2>&1
for r in ours cudnn; do ncu -i $OUT/$r.ncu-rep --page raw --csv > $OUT/${r}_raw.csv 2>&1; done
ncu -i $OUT/ours.ncu-rep --page source --csv > $OUT/ours_source.csv 2>&1
timeout 300 python tools/attn_library.py --out $OUT/library.json > $OUT/library.log 2>&1
ls -la $OUT
