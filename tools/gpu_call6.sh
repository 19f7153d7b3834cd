#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py > $OUT/build6.log 2>&1
timeout 600 python tools/packets_bench.py --M 400 800 1200 1600 2000 --t 2 3 4 5 6 > $OUT/packets_bench6.txt 2>&1
timeout 300 python tools/quick_bench.py --m 7 8 > $OUT/quick78.txt 2>&1
timeout 1500 python tools/tune_shapes.py run packets > $OUT/tune_pkt6.txt 2>&1
HAMMING_LIB=tune_libs/probe.so timeout 600 python tools/power_probe.py --probe --only6 > $OUT/power6.txt 2>&1
cat $OUT/packets_bench6.txt $OUT/quick78.txt $OUT/power6.txt
