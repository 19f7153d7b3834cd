#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py > $OUT/build12.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "long or smoke" > $OUT/pytest12.log 2>&1
tail -2 $OUT/pytest12.log
timeout 900 python tools/tune_shapes.py run long > $OUT/tune_long12.txt 2>&1
cat $OUT/tune_long12.txt
timeout 1500 compute-sanitizer --tool initcheck --print-limit 100000 python tools/sanitize_workload.py --initcheck > $OUT/initcheck12.txt 2>&1
echo "rc=$?" >> $OUT/initcheck12.txt
tail -4 $OUT/initcheck12.txt
