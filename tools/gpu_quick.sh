#!/bin/bash
# Quick GPU iteration: build, GPU tests, smoke, timeline, bench without CPU leg.
#   gpurun --timeout 1500 -- bash tools/gpu_quick.sh <tag> [notest]
OUT=gpurun_out/${1:-quick}
mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
if [ "$2" != notest ]; then
  timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  tail -5 $OUT/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
tail -2 $OUT/smoke.log
timeout 300 python tools/timeline.py > $OUT/timeline.txt 2>&1; tail -1 $OUT/timeline.txt
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
tail -c 600 $OUT/bench.log
