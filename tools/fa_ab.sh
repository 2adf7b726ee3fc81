#!/bin/bash
# FA variant A/B on one box: parity tests, then interleaved timings.
OUT=gpurun_out/${1:-fa_ab}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k attention > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
DS_FA_CHUNK=0 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k attention > $OUT/pytest_old.log 2>&1; echo "rc=$?" >> $OUT/pytest_old.log
for r in 0 1 2; do
  for c in 0 1; do echo "chunk=$c $(DS_FA_CHUNK=$c python tools/attn_bench.py)"; done
done > $OUT/chunk.txt 2>&1
python tools/ab_run.py --rounds 3 --cmd "python tools/attn_bench.py" ab/emu2.so ab/emu3.so ab/emu4.so ab/emu8.so > $OUT/emu.txt 2>&1
