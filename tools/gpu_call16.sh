#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py > $OUT/build16.log 2>&1
for mt in "400 5" "800 6" "2000 3"; do
  set -- $mt
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:packets_decode -s 1 -c 1 \
    -o $OUT/pk16_$1_$2 -f python tools/packets_prof.py $1 $2 > $OUT/pk16_$1_$2.log 2>&1
done
ls $OUT/pk16*
