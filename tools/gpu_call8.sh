#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python tools/tune_shapes.py run power6 > $OUT/power6_wait.txt 2>&1
cat $OUT/power6_wait.txt
