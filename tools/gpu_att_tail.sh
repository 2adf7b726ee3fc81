#!/bin/bash
# Stand-alone attention tail (merge release fence, merge loop): parity of ab/att_new.so,
# same-box A/B against ab/att_head.so (decode-like anchor chain, 1 and 8 rows), and
# stamp timelines (ab/att_stamp*.so, one launch's phases; DS_ATT_PREFETCH=16 skips the softmax).
OUT=gpurun_out/${1:-att_tail}
mkdir -p $OUT
DS_LIB=ab/att_new.so timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_batch.py tests/test_gpu_parity.py -q -x > $OUT/pytest.log 2>&1
echo "rc=$?" >> $OUT/pytest.log; tail -3 $OUT/pytest.log
for r in 0 1; do for L in att_head att_new; do for b in 0 8; do
  echo "$L b=$b $(DS_LIB=ab/$L.so timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-90)"
done; done; done > $OUT/ab.txt 2>&1
cat $OUT/ab.txt
DS_LIB=ab/att_stamp.so timeout 300 python tools/anchor_alone.py --reps 1 > $OUT/stamp_new.txt 2>&1
DS_LIB=ab/att_stamp_head.so timeout 300 python tools/anchor_alone.py --reps 1 > $OUT/stamp_head.txt 2>&1
DS_ATT_PREFETCH=16 DS_LIB=ab/att_stamp.so timeout 300 python tools/anchor_alone.py --reps 1 > $OUT/stamp_nosoftmax.txt 2>&1
DS_ATT_PREFETCH=10 DS_LIB=ab/att_stamp.so timeout 300 python tools/anchor_alone.py --reps 1 > $OUT/stamp_nomath.txt 2>&1
ls -la $OUT
# batch leg of the bench in isolation vs anchor_alone (HEAD library), and with x streaming off
for x in 1 0; do
  DS_GEMVB_XSTREAM=$x timeout 600 python tools/batch_leg_probe.py > $OUT/leg_xs$x.txt 2>&1
  tail -1 $OUT/leg_xs$x.txt
done
for b in 4 8; do echo "alone b=$b $(timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-90)"; done > $OUT/alone.txt 2>&1
cat $OUT/alone.txt
