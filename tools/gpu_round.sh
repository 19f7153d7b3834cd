#!/bin/bash
# One GPU session: bench (default C5), launch list, one ncu --set full capture
# of the decode kernel, and the GPU test suite.  Outputs land in gpurun_out/.
set -x
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $OUT/gpu_info.csv
python __graft_entry__.py > $OUT/build.log 2>&1
timeout 900 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.log
for c in c3m6 c3m5 c3m4 c3m3 c4; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.log
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_launch_bench.log 2>&1
for m in 6 5 4 3; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiles_kernel -s 3 -c 1 \
    -o $OUT/prof_m$m -f python bench.py --config c3m$m --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_full_m$m.log 2>&1
done
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
tail -3 $OUT/pytest_gpu.log
