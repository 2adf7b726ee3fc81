#!/bin/bash
OUT=gpurun_out/${1:-att_items}
mkdir -p $OUT
for it in 148 222 296 444 592; do for b in 0 8; do
  echo "items=$it b=$b $(DS_ATT_ITEMS=$it timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-90)"
done; done > $OUT/items.txt 2>&1
cat $OUT/items.txt
