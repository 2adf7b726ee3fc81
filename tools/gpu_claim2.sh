#!/bin/bash
# Claimed tiles in the batched GEMV too: GPU suite, then same-box A/B (DS_GEMV_CLAIM only gates the
# single-row kernel; the batched A/B is against ab/claim_head.so = HEAD).
OUT=gpurun_out/${1:-claim2}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log
cp paper_2411_02820_b200/libdroidspeak.so ab/claim_new.so
for r in 0 1; do for L in claim_head claim_new; do for b in 0 4 8; do
  echo "$L b=$b $(DS_LIB=ab/$L.so timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-90)"
done; done; done > $OUT/ab.txt 2>&1
cat $OUT/ab.txt
