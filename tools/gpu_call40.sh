#!/bin/bash
OUT=gpurun_out
python __graft_entry__.py > $OUT/build40.log 2>&1
for r in 1 2; do
for lib in default tune_libs/dyn_2.so tune_libs/dyn_4.so tune_libs/dyn_0.so; do
  if [ $lib = default ]; then unset HAMMING_LIB; else export HAMMING_LIB=$lib; fi
  python tools/quick_bench.py --m 3 4 5 6 --gib 0.25 --reps 20 --tag $lib 2>&1 | grep "syn=True"
done
done
