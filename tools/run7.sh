bash tools/gpu_check.sh r01e quick
OUT=gpurun_out/r01e
timeout 600 python -m pytest tests/test_gpu_quality.py -x -q -s > $OUT/pytest_quality.log 2>&1; echo "rc=$?" >> $OUT/pytest_quality.log
