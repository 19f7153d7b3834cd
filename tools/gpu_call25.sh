#!/bin/bash
OUT=gpurun_out
python __graft_entry__.py > $OUT/build25.log 2>&1
python __graft_entry__.py smoke > $OUT/smoke25.log 2>&1; tail -1 $OUT/smoke25.log
timeout 1200 python -m pytest tests -m gpu -q -x -k "parity or shards or adt or fullsize or secded or smoke" > $OUT/pytest25.log 2>&1
tail -2 $OUT/pytest25.log
python tools/small_call_probe.py > $OUT/small25.txt 2>&1; cat $OUT/small25.txt
timeout 300 python tools/small_packets.py > $OUT/small_packets25.txt 2>&1; tail -30 $OUT/small_packets25.txt
