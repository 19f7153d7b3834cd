#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py > $OUT/build20.log 2>&1
timeout 2400 python tools/pkt_shape_sweep.py tune_libs/pkt_tune.so > $OUT/pkt_sweep21.txt 2>&1
