#!/bin/bash
# Why the bench's batch-leg decode is slower than the same leg alone: probe as-is, probe after a
# fragmenting allocation pattern, and the bench with only the 8-row batch leg.
OUT=gpurun_out/${1:-leg_var}
mkdir -p $OUT
timeout 600 python tools/batch_leg_probe.py --sizes 8 > $OUT/probe.txt 2>&1; tail -1 $OUT/probe.txt
timeout 600 python tools/batch_leg_probe.py --sizes 8 --fragment-gb 40 > $OUT/probe_frag.txt 2>&1; tail -1 $OUT/probe_frag.txt
timeout 1200 python bench.py --steps 10 --warmup 3 --batch-leg 8 --no-cpu-baseline > $OUT/bench.txt 2>&1
python -c "
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith('{\"metric\"')][-1]
print(json.dumps(json.loads(l)['batch']))
" $OUT/bench.txt > $OUT/bench_batch.txt 2>&1
cat $OUT/bench_batch.txt
