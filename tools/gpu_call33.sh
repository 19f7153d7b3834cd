#!/bin/bash
OUT=gpurun_out
python __graft_entry__.py > $OUT/build33.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > $OUT/pytest33.log 2>&1
tail -3 $OUT/pytest33.log
timeout 1200 compute-sanitizer --tool initcheck --print-limit 100 python tools/sanitize_workload.py --initcheck > $OUT/initcheck33.txt 2>&1
echo "rc=$?" >> $OUT/initcheck33.txt; tail -3 $OUT/initcheck33.txt
