#!/bin/bash
# packet tests + the paper-grid bench after a packet-decoder change -> profiles/r02e_packets_bench.txt
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_packets.py tests/test_boundary_cpu.py -x -q > $OUT/pkc_pytest.log 2>&1; echo "rc=$?" >> $OUT/pkc_pytest.log; tail -2 $OUT/pkc_pytest.log
python __graft_entry__.py smoke 2>&1 | tail -1
timeout 600 python tools/packets_bench.py --M 400 800 1200 1600 2000 --t 2 3 4 5 6 > $OUT/pkc_grid.txt 2>&1; cat $OUT/pkc_grid.txt
