#!/bin/bash
OUT=gpurun_out
python __graft_entry__.py > $OUT/build35.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=8 > $OUT/pytest35.log 2>&1
tail -12 $OUT/pytest35.log
