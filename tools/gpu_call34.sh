#!/bin/bash
OUT=gpurun_out
python __graft_entry__.py > $OUT/build34.log 2>&1
timeout 300 python tools/small_packets.py > $OUT/small_packets34.txt 2>&1; tail -16 $OUT/small_packets34.txt
timeout 900 python bench.py --steps 3 --no-e2e --no-cpu > $OUT/bench34.json 2> $OUT/bench34.log
python -c "
import json
d=json.loads(open('$OUT/bench34.json').read().strip().splitlines()[-1])
print([ (p['coded_bytes'],p['cold_us'],p['warm_us']) for p in d['sweeps']['c2_packet_size_15_11']['points']])"
