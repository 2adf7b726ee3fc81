#!/bin/bash
OUT=gpurun_out/${1:-fa_emu}
mkdir -p $OUT
for r in 0 1; do for v in main fa_emu2 fa_emu3 fa_emu8; do
  if [ $v = main ]; then L=""; else L="ab/$v.so"; fi
  echo "$v $(DS_LIB=$L timeout 120 python tools/attn_bench.py 2>&1 | tail -1)"
done; done > $OUT/emu.txt 2>&1
cat $OUT/emu.txt
