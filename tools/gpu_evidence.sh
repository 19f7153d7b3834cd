#!/bin/bash
# Evidence session for a round: build + smoke, launch list and DRAM bytes of the bench's own decode
# launch, one --set full capture, sanitizers, the GPU tests and the default bench.  -> gpurun_out/
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py smoke > $OUT/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/${TAG}_smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches_c5.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-sweeps > $OUT/${TAG}_launch_bench.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:tiles_kernel -s 4 -c 1 --csv --log-file $OUT/${TAG}_dram_c5.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-sweeps > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiles_kernel -s 4 -c 1 \
  -o $OUT/${TAG}_full_m6 -f python bench.py --config c3m6 --steps 1 --warmup 3 --no-e2e --no-cpu --no-sweeps \
  > $OUT/${TAG}_full_m6.log 2>&1
for tool in ${SANITIZERS:-}; do  # compute-sanitizer is closed on the pool (exit 86); opt in with SANITIZERS="initcheck memcheck"
  echo "== $tool" >> $OUT/${TAG}_sanitizer.txt
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_workload.py $([ $tool = initcheck ] && echo --initcheck) \
    >> $OUT/${TAG}_sanitizer.txt 2>&1
  echo "rc=$?" >> $OUT/${TAG}_sanitizer.txt
done
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.log
sleep 5
timeout 900 python bench.py > $OUT/${TAG}_bench_c5.json 2> $OUT/${TAG}_bench_c5.log
timeout 600 python bench.py --impl reference > $OUT/${TAG}_bench_reference.json 2> $OUT/${TAG}_bench_reference.log
tail -3 $OUT/${TAG}_pytest_gpu.log; tail -8 $OUT/${TAG}_sanitizer.txt; head -c 1500 $OUT/${TAG}_bench_c5.json
