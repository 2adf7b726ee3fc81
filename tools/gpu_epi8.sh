#!/bin/bash
# Same-box A/B of the pair GEMM's epilogue warps (DS_GEMM_EPI_WARPS=4|8):
# per-shape GEMM times, the o-proj epilogue probe, the consumer step, then the GPU tests.
OUT=gpurun_out/${1:-epi8}; mkdir -p $OUT
for ew in 4 8; do
  DS_GEMM_EPI_WARPS=$ew timeout 300 python tools/oproj_epi_probe.py > $OUT/probe_$ew.txt 2>&1
  DS_GEMM_EPI_WARPS=$ew timeout 300 python tools/gemm_bench.py > $OUT/gemm_$ew.txt 2>&1
done
for r in 1 2 3; do for ew in 4 8; do
  echo "ew=$ew round=$r: $(DS_GEMM_EPI_WARPS=$ew timeout 300 python tools/step_time.py --steps 30 2>&1 | tail -1)" >> $OUT/step.txt
done; done
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/gputest.log 2>&1; echo "rc=$?" >> $OUT/gputest.log
