#!/bin/bash
# In-step A/B of FA variants (power-capped consumer step): variant 1 vs 3 vs 3 with 1-in-8 emulation.
OUT=gpurun_out/${1:-fa_step}
mkdir -p $OUT
for r in 0 1 2; do
  echo "v1   $(DS_FA_VARIANT=1 timeout 300 python tools/step_time.py 2>&1 | tail -1)"
  echo "v3   $(DS_FA_VARIANT=3 timeout 300 python tools/step_time.py 2>&1 | tail -1)"
  echo "v3e8 $(DS_LIB=ab/fa_emu8.so DS_FA_VARIANT=3 timeout 300 python tools/step_time.py 2>&1 | tail -1)"
done > $OUT/step.txt 2>&1
cat $OUT/step.txt
