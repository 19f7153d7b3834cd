#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python __graft_entry__.py > $OUT/build3.log 2>&1
for mt in "400 5" "2000 2"; do
  set -- $mt
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:packets_decode -s 1 -c 1 \
    -o $OUT/pk_$1_$2 -f python tools/packets_prof.py $1 $2 > $OUT/pk_$1_$2.log 2>&1
done
timeout 600 python tools/adt_eq1.py --out $OUT/r02_adt_eq1.md > $OUT/adt_eq1.txt 2>&1
ls -la $OUT
