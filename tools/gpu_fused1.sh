#!/bin/bash
# fused packet decoder: correctness, grid bench, shape sweep (tuning build)
OUT=gpurun_out
mkdir -p $OUT tune_libs
timeout 900 python -m pytest tests/test_gpu_packets.py -x -q > $OUT/f1_pytest.log 2>&1; echo "rc=$?" >> $OUT/f1_pytest.log
tail -15 $OUT/f1_pytest.log
timeout 600 python tools/packets_bench.py --M 400 800 1200 1600 2000 --t 2 3 4 5 6 > $OUT/f1_grid.txt 2>&1
cat $OUT/f1_grid.txt
timeout 1200 python tools/fused_sweep.py tune_libs/fused_tune.so 400 5 400 2 800 6 1200 2 2000 3 > $OUT/f1_sweep.txt 2>&1
cat $OUT/f1_sweep.txt | grep -v "^  L="
