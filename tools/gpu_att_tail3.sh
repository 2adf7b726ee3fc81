#!/bin/bash
# Stand-alone attention round 3: stream-per-warp P.V with the full-piece fast path (ab/att_pvs3.so, the
# new default) vs the lane-layout P.V (ab/att_lanes.so) and HEAD; whole GPU suite on the new default.
OUT=gpurun_out/${1:-att_tail3}
mkdir -p $OUT
DS_LIB=ab/att_pvs3.so timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_pvs3.log 2>&1
echo "rc=$?" >> $OUT/pytest_pvs3.log; tail -2 $OUT/pytest_pvs3.log
for r in 0 1; do for L in att_head att_lanes att_pvs3; do for b in 0 4 8; do
  echo "$L b=$b $(DS_LIB=ab/$L.so timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-90)"
done; done; done > $OUT/ab.txt 2>&1
cat $OUT/ab.txt
DS_LIB=ab/att_pvs3_stamp.so timeout 300 python tools/anchor_alone.py --reps 1 > $OUT/stamp_pvs3.txt 2>&1
ls -la $OUT
