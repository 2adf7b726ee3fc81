#!/bin/bash
# ncu evidence for the consumer step (BASELINE config 2): launch list of one
# step, then full captures of the pair GEMMs (layer 26: QKV, o-proj, W1, W2),
# one FA launch and the persistent anchor.
#   gpurun --timeout 2400 -- bash tools/prof_step.sh <tag>
OUT=gpurun_out/${1:-prof}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_partial.csv python tools/profile_step.py --what partial > $OUT/ncu_launch.log 2>&1
NCU="ncu --profile-from-start off --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:gemm_tc2 -c 4 -o $OUT/prof_gemm python tools/profile_step.py --what partial > $OUT/ncu_gemm.log 2>&1
timeout 600 $NCU -k regex:"fa_(tc|dual)" -c 1 -o $OUT/prof_fa python tools/profile_step.py --what partial > $OUT/ncu_fa.log 2>&1
timeout 600 $NCU -k regex:anchor_persistent -c 1 -o $OUT/prof_anchor python tools/profile_step.py --what partial > $OUT/ncu_anchor.log 2>&1
ls -la $OUT
# the stand-alone anchor kernels (single stream): TMA-staged GEMV and split-KV attention
timeout 600 $NCU -k regex:"gemv_tma|attn_decode" -c 5 -o $OUT/prof_anchor_launch python tools/profile_step.py --what partial --single > $OUT/ncu_anchor_launch.log 2>&1
