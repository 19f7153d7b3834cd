#!/bin/bash
OUT=gpurun_out
python __graft_entry__.py > $OUT/build23.log 2>&1
python tools/small_call_probe.py > $OUT/small23.txt 2>&1
ncu --metrics gpu__time_duration.sum --csv python tools/small_call_probe.py > $OUT/small23_ncu.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:perfect_long -s 2 -c 1 \
    -o $OUT/long7 -f python tools/quick_bench.py --m 7 --reps 1 > $OUT/long7.log 2>&1
cat $OUT/small23.txt; grep -c tiles_kernel $OUT/small23_ncu.csv
