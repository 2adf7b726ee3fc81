#!/bin/bash
# Same-box A/B of ab/fa_head.so vs ab/$2.so: attention kernel alone, then the consumer step.
OUT=gpurun_out/${1:-fa_ab}; V=${2}
mkdir -p $OUT
DS_LIB=ab/$V.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for r in 0 1; do for L in fa_head $V; do echo "$L $(DS_LIB=ab/$L.so timeout 120 python tools/attn_bench.py 2>&1 | tail -1)"; done; done > $OUT/ab.txt 2>&1
for r in 0 1 2; do for L in fa_head $V; do echo "$L $(DS_LIB=ab/$L.so timeout 300 python tools/step_time.py 2>&1 | tail -1)"; done; done >> $OUT/ab.txt 2>&1
cat $OUT/ab.txt
