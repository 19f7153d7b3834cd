#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py > $OUT/build7.log 2>&1
for mt in "1600 3" "400 6" "2000 2"; do
  set -- $mt
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:packets_decode -s 1 -c 1 \
    -o $OUT/pk7_$1_$2 -f python tools/packets_prof.py $1 $2 > $OUT/pk7_$1_$2.log 2>&1
done
timeout 1200 python tools/tune_shapes.py run power6 > $OUT/power6_shapes.txt 2>&1
cat $OUT/power6_shapes.txt
