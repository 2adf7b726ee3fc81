#!/bin/bash
# Pair-GEMM raster / L2-policy sweep: event times and ncu DRAM bytes per launch for
# the recompute shapes (tools/gemm_bench.py), one process per setting.
#   bash tools/raster_sweep.sh "DS_GEMM_GROUP=8 DS_GEMM_GROUP=16 ..."   (settings: VAR=val[,VAR=val])
#   -> gpurun_out/raster_<i>.{txt,csv}
i=0
for cfg in ${1:-DS_GEMM_GROUP=8 DS_GEMM_GROUP=16}; do
  envs=$(echo "$cfg" | tr ',' ' ')
  echo "$cfg" > gpurun_out/raster_time_$i.txt
  env $envs python tools/gemm_bench.py >> gpurun_out/raster_time_$i.txt 2>&1
  env $envs ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
    --clock-control none -k regex:gemm --csv --log-file gpurun_out/raster_$i.csv python tools/gemm_bench.py > /dev/null 2>&1
  i=$((i+1))
done
