#!/bin/bash
# Stand-alone attention round 2: merge (one-thread acq_rel fences, explicit shared loads, interleaved
# chains) in ab/att_new2.so; stream-per-warp P.V in ab/att_pvs2.so.  Parity of both, same-box A/B
# against ab/att_head.so, stamp timelines with the P.V phase's SM cycles.
OUT=gpurun_out/${1:-att_tail2}
mkdir -p $OUT
for L in att_new2 att_pvs2; do
  DS_LIB=ab/$L.so timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_batch.py tests/test_gpu_parity.py tests/test_gpu_quality.py -q -x > $OUT/pytest_$L.log 2>&1
  echo "rc=$?" >> $OUT/pytest_$L.log; tail -2 $OUT/pytest_$L.log
done
for r in 0 1; do for L in att_head att_new2 att_pvs2; do for b in 0 8; do
  echo "$L b=$b $(DS_LIB=ab/$L.so timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-90)"
done; done; done > $OUT/ab.txt 2>&1
cat $OUT/ab.txt
DS_LIB=ab/att_stamp2.so timeout 300 python tools/anchor_alone.py --reps 1 > $OUT/stamp_new2.txt 2>&1
DS_LIB=ab/att_pvs_stamp2.so timeout 300 python tools/anchor_alone.py --reps 1 > $OUT/stamp_pvs2.txt 2>&1
ls -la $OUT
