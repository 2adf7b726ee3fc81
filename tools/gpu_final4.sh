#!/bin/bash
# End-of-round evidence (tools/gpu_profiles_r02.sh) plus the batch leg alone after it.
bash tools/gpu_profiles_r02.sh ${1:-r02_final4}
OUT=gpurun_out/${1:-r02_final4}
timeout 600 python tools/batch_leg_probe.py > $OUT/batch_leg_probe.txt 2>&1
tail -1 $OUT/batch_leg_probe.txt
for b in 0 4 8; do echo "alone b=$b $(timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-90)"; done > $OUT/alone.txt 2>&1
cat $OUT/alone.txt
