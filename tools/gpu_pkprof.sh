#!/bin/bash
# ncu --set full of the packet decoder at the weakest cells of the paper grid -> gpurun_out/pk_<M>_<t>.ncu-rep
OUT=gpurun_out
mkdir -p $OUT
for cell in ${CELLS:-"400 5" "400 2"}; do
  set -- $cell
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:packets_decode -s 1 -c 1 \
    -o $OUT/pk_${1}_${2} -f python tools/packets_prof.py $1 $2 > $OUT/pk_ncu_${1}_${2}.log 2>&1
done
timeout 300 python tools/packets_bench.py --M 400 --t 2 3 4 5 6 > $OUT/pk_grid400.txt 2>&1; cat $OUT/pk_grid400.txt
