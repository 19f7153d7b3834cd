#!/bin/bash
for r in 1 2 3; do
  for lib in default tune_libs/dyn34_4.so tune_libs/dyn34_16.so tune_libs/dyn34_64.so; do
    if [ $lib = default ]; then unset HAMMING_LIB; else export HAMMING_LIB=$lib; fi
    python tools/quick_bench.py --m 3 4 --gib 0.25 --reps 20 --tag $lib 2>&1 | grep "syn=True"
  done
done
