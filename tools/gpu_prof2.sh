#!/bin/bash
# Profiling session: packets kernel (source-level), small-m decode without syndromes, copy ceiling.
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py > $OUT/build2.log 2>&1
timeout 300 python tools/copy_ceiling.py --mib 256 2048 > $OUT/copy_ceiling.jsonl 2>&1
timeout 600 python tools/packets_bench.py --M 400 800 1200 1600 2000 --t 2 3 4 5 6 > $OUT/packets_bench.txt 2>&1
timeout 300 python tools/packets_bench.py --M 400 2000 --t 2 5 --P 2097152 > $OUT/packets_bench_2m.txt 2>&1
for mt in "400 5" "2000 2" "800 4"; do
  set -- $mt
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:packets_decode -s 2 -c 1 \
    -o $OUT/pk_$1_$2 -f python tools/packets_prof.py $1 $2 > $OUT/pk_$1_$2.log 2>&1
done
for m in 3 4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tiles_kernel -s 4 -c 1 \
    -o $OUT/nosyn_m$m -f python bench.py --config c3m$m --steps 1 --warmup 3 --no-e2e --no-cpu --no-syndromes --no-sweeps \
    > $OUT/nosyn_m$m.log 2>&1
done
ls -la $OUT
