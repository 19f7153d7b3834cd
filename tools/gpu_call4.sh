#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py > $OUT/build4.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest4.log 2>&1
tail -3 $OUT/pytest4.log
timeout 300 python tools/quick_bench.py --m 3 4 5 6 > $OUT/quick4.txt 2>&1
cat $OUT/quick4.txt
timeout 300 python tools/packets_overhead.py 400 5 > $OUT/pk_over_400_5.txt 2>&1
timeout 300 python tools/packets_overhead.py 2000 2 > $OUT/pk_over_2000_2.txt 2>&1
cat $OUT/pk_over_*.txt
timeout 600 python bench.py --config c3m3 --steps 5 --no-e2e --no-cpu --no-sweeps > $OUT/c3m3.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/pk_launches.csv python tools/packets_overhead.py 400 5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiles_kernel -s 4 -c 1 \
    -o $OUT/m3pair -f python bench.py --config c3m3 --steps 1 --warmup 3 --no-e2e --no-cpu --no-sweeps > $OUT/m3pair.log 2>&1
