#!/bin/bash
OUT=gpurun_out
python __graft_entry__.py > $OUT/build24.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:tiles_kernel -s 5 -c 1 -o $OUT/small24 -f python tools/small_call_probe.py > $OUT/small24.log 2>&1
timeout 600 ncu --set full --cache-control none --import-source on -k regex:tiles_kernel -s 5 -c 1 -o $OUT/small24w -f python tools/small_call_probe.py > $OUT/small24w.log 2>&1
