#!/bin/bash
# ncu evidence for the current build (one GPU): launch list of the default bench,
# DRAM bytes of the C5 decode launch, and a --set full capture of the decode
# kernel for each m at C3 (256 MiB).  Writes gpurun_out/prof_<tag>_*.
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches_c5.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $OUT/${TAG}_launch_bench.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:tiles_kernel -s 4 -c 1 --csv --log-file $OUT/${TAG}_dram_c5.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
for m in 6 5 4 3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiles_kernel -s 4 -c 1 \
    -o $OUT/${TAG}_full_m$m -f python bench.py --config c3m$m --steps 1 --warmup 3 --no-e2e --no-cpu \
    > $OUT/${TAG}_full_m$m.log 2>&1
done
ls -la $OUT | grep $TAG
