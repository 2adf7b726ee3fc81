OUT=gpurun_out/att1; mkdir -p $OUT
python -m paper_2411_02820_b200._build > $OUT/build.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"attn_decode_tma" -c 2 -o $OUT/prof python tools/anchor_alone.py --profile > $OUT/ncu.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --cache-control none --csv --log-file $OUT/launches.csv python tools/anchor_alone.py --profile > $OUT/ncu_launch.log 2>&1
ls $OUT
