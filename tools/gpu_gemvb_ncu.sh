#!/bin/bash
# ncu --set full of one W1 GEMV launch: single-row TMA kernel vs batched (4 rows).
OUT=gpurun_out/${1:-gemvb_ncu}
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemv_tma_kernel" -s 2 -c 1 -o $OUT/single python tools/anchor_alone.py --reps 1 > $OUT/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemv_batch_kernel" -s 2 -c 1 -o $OUT/batch python tools/anchor_alone.py --batch 4 --reps 1 > $OUT/ncu2.log 2>&1
for r in single batch; do
  ncu -i $OUT/$r.ncu-rep --page source --csv > $OUT/${r}_source.csv 2>&1
  ncu -i $OUT/$r.ncu-rep --page raw --csv > $OUT/${r}_raw.csv 2>&1
done
ls -la $OUT
