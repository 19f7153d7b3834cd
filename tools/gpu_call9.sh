#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py > $OUT/build9.log 2>&1
HAMMING_LIB=tune_libs/probe.so timeout 600 python tools/power_probe.py --probe --only6 > $OUT/power9.txt 2>&1
timeout 600 python tools/packets_bench.py --M 400 800 1200 1600 2000 --t 2 3 4 5 6 > $OUT/packets_bench9.txt 2>&1
cat $OUT/power9.txt $OUT/packets_bench9.txt
