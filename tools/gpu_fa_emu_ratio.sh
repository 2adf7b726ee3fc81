#!/bin/bash
# Dual FA exp-emulation ratio A/B (profiles/r02_fa_emu_ratio_ab.txt).  Build the variants first (CPU box):
#   bash tools/variant_build.sh emu8 ""; bash tools/variant_build.sh emu0 -DDS_FA_DUAL_EMU=0
#   bash tools/variant_build.sh emu16 -DDS_FA_DUAL_EMU=16
OUT=gpurun_out/emu_ab; mkdir -p $OUT
python tools/ab_run.py --rounds 3 --cmd "timeout 120 python tools/attn_bench.py" ab/emu8.so ab/emu0.so ab/emu16.so > $OUT/attn.txt 2>&1
python tools/ab_run.py --rounds 3 --cmd "timeout 300 python tools/step_time.py --steps 30" ab/emu8.so ab/emu0.so ab/emu16.so > $OUT/step.txt 2>&1
