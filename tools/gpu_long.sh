#!/bin/bash
# long codes (m = 7, 8): parity tests, then A/B of the in-place ring (default build) against the
# previous two-buffer kernel (tune_libs/base.so) -> gpurun_out/long.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "long" 2>&1 | tail -2
for r in 1 2; do
  for lib in default tune_libs/base.so; do
    if [ $lib = default ]; then unset HAMMING_LIB; else export HAMMING_LIB=$lib; fi
    python tools/quick_bench.py --m 7 8 --gib 2 --reps 8 --tag $lib 2>&1 | grep "Gbit"
    python tools/quick_bench.py --m 7 8 --gib 0.25 --reps 20 --tag "$lib 256MiB" 2>&1 | grep "Gbit"
  done
done
