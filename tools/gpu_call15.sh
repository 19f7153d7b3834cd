#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py > $OUT/build15.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "packets or smoke" > $OUT/pytest15.log 2>&1
tail -2 $OUT/pytest15.log
timeout 600 python tools/packets_bench.py --M 400 800 1200 1600 2000 --t 2 3 4 5 6 > $OUT/packets_bench15.txt 2>&1
cat $OUT/packets_bench15.txt
