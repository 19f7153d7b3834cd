#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_packets.py -x -q > $OUT/f4_pytest.log 2>&1; echo "rc=$?" >> $OUT/f4_pytest.log
tail -3 $OUT/f4_pytest.log
timeout 1500 python tools/fused_sweep.py tune_libs/fused_tune.so 400 5 400 2 800 6 1200 2 2000 3 1600 3 > $OUT/f4_sweep.txt 2>&1
cat $OUT/f4_sweep.txt | grep -v "^  L="
