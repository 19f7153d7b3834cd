#!/bin/bash
# A/B of (63,57) launch shapes on the sustained C5 bench, alternating, same box.
OUT=gpurun_out
python __graft_entry__.py > $OUT/build_ab.log 2>&1
for r in 1 2 3; do
  for lib in default tune_libs/c5_w4_s3.so tune_libs/c5_w12_s2.so tune_libs/c5_w6_s3.so; do
    if [ $lib = default ]; then unset HAMMING_LIB; else export HAMMING_LIB=$lib; fi
    sleep 3
    python bench.py --no-e2e --no-cpu --no-sweeps 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks'].get('power_w'), d['config']['grid_blocks'])"
  done
done
