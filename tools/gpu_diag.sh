#!/bin/bash
# Diagnostics: batch decode diff, pipe-rate probe, FA ncu source capture.
OUT=gpurun_out/${1:-diag}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 300 python tools/batch_debug.py > $OUT/batch_debug.txt 2>&1; cat $OUT/batch_debug.txt | tail -20
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_probe tools/pipe_probe.cu && timeout 120 /tmp/pipe_probe > $OUT/pipe_probe.txt 2>&1; cat $OUT/pipe_probe.txt
bash tools/ncu_fa.sh ${1:-diag}/fa > /dev/null 2>&1; ls $OUT/fa
