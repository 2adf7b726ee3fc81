#!/bin/bash
OUT=gpurun_out/${1:-gemvb_ks}
mkdir -p $OUT
for r in 0 1; do for ks in 4096 2048 1024; do for b in 2 4 8; do
  echo "ks=$ks b=$b $(DS_GEMVB_KS=$ks timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-100)"
done; done; done > $OUT/times.txt 2>&1
cat $OUT/times.txt
