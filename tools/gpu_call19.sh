#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py > $OUT/build19.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:packets_decode -s 1 -c 1 \
    -o $OUT/pk19_400_5 -f python tools/packets_prof.py 400 5 > $OUT/pk19.log 2>&1
