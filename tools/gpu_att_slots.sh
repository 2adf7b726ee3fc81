#!/bin/bash
OUT=gpurun_out/${1:-att_slots}
mkdir -p $OUT
for sl in 8 10 12 14 16; do for b in 0 8; do
  echo "slots=$sl b=$b $(DS_ATT_SLOTS=$sl timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-90)"
done; done > $OUT/slots.txt 2>&1
cat $OUT/slots.txt
