#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py > $OUT/build11.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "packets or smoke" > $OUT/pytest11.log 2>&1
tail -2 $OUT/pytest11.log
timeout 600 python tools/packets_bench.py --M 400 800 1200 1600 2000 --t 2 3 4 5 6 > $OUT/packets_bench11.txt 2>&1
cat $OUT/packets_bench11.txt
timeout 1500 compute-sanitizer --tool initcheck --print-limit 1000000 python tools/sanitize_workload.py > $OUT/initcheck11.txt 2>&1
echo "rc=$?" >> $OUT/initcheck11.txt
grep -c "Uninitialized" $OUT/initcheck11.txt
