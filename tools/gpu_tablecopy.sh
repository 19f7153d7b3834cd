#!/bin/bash
# A/B: the 64 KB CTA tables by one TMA bulk copy (default build) vs the thread copy loop (tune_libs/base.so)
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_secded.py -x -q -k "m4 or m5 or 4 or 5" > $OUT/tc_pytest.log 2>&1; echo "rc=$?" >> $OUT/tc_pytest.log; tail -2 $OUT/tc_pytest.log
for m in 4 5; do HAMMING_LIB=build/tune/timing.so python tools/timing_probe.py $m 256 | tail -2; done
for r in 1 2; do
  for lib in base default; do
    if [ $lib = default ]; then unset HAMMING_LIB; else export HAMMING_LIB=tune_libs/base.so; fi
    python tools/quick_bench.py --m 3 4 5 6 --gib 0.25 --reps 20 --tag $lib 2>&1 | grep "syn=True"
    python tools/quick_bench.py --m 4 5 --gib 0.25 --reps 20 --secded --tag $lib 2>&1 | grep "syn=True\|flags"
  done
done
