#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py > $OUT/build5.log 2>&1
timeout 900 python tools/tune_shapes.py run m3 > $OUT/tune_m3.txt 2>&1
timeout 600 python tools/packets_bench.py --M 400 800 1200 1600 2000 --t 2 3 4 5 6 > $OUT/packets_bench5.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "packets or smoke" > $OUT/pytest5.log 2>&1
tail -2 $OUT/pytest5.log
cat $OUT/tune_m3.txt $OUT/packets_bench5.txt
