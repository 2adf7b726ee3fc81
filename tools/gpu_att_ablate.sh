#!/bin/bash
# Stand-alone attention: chain of attention launches only (DS_ABLATE_ANCHOR=29), with the
# scores / P.V math skipped (DS_ATT_PREFETCH bits, timing only), single row and 8 rows.
OUT=gpurun_out/${1:-att_ablate}
mkdir -p $OUT
for pf in 0 2 8 10; do for b in 0 8; do
  echo "prefetch=$pf b=$b $(DS_ABLATE_ANCHOR=29 DS_ATT_PREFETCH=$pf timeout 300 python tools/anchor_alone.py --batch $b --reps 10 2>&1 | tail -1 | cut -c1-80)"
done; done > $OUT/ablate.txt 2>&1
cat $OUT/ablate.txt
