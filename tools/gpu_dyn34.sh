#!/bin/bash
# A/B of the dynamic tail rounds for m = 3, 4 (tune_libs/dyn34_<d>.so: -DHAM_DYN3=d -DHAM_DYN4=d) -> profiles/r02_dyn_tail_m34.txt
for r in 1 2 3; do
  for lib in default tune_libs/dyn34_4.so tune_libs/dyn34_16.so tune_libs/dyn34_64.so; do
    if [ $lib = default ]; then unset HAMMING_LIB; else export HAMMING_LIB=$lib; fi
    python tools/quick_bench.py --m 3 4 --gib 0.25 --reps 20 --tag $lib 2>&1 | grep "syn=True"
  done
done
