#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
for cell in "400 5" "2000 3"; do
  set -- $cell
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:packets_fused -s 1 -c 1 \
    -o $OUT/f2_${1}_${2} -f python tools/packets_prof.py $1 $2 > $OUT/f2_ncu_${1}_${2}.log 2>&1
done
timeout 1200 python tools/fused_sweep.py tune_libs/fused_tune.so 400 5 2000 3 > $OUT/f2_sweep.txt 2>&1
cat $OUT/f2_sweep.txt | grep -v "^  L="
