#!/bin/bash
# Quick state check on a fresh box: smoke, the GPU tests, the default bench.  -> gpurun_out/
TAG=${1:-r02d}
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/${TAG}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
sleep 5
timeout 900 python bench.py > $OUT/${TAG}_bench_c5.json 2> $OUT/${TAG}_bench_c5.log
tail -2 $OUT/${TAG}_smoke.log; tail -3 $OUT/${TAG}_pytest_gpu.log; head -c 1200 $OUT/${TAG}_bench_c5.json
