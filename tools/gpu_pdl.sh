#!/bin/bash
# A/B of programmatic dependent launch for small calls (tune_libs/nopdl.so: -DHAM_SMALL_PDL=0) -> profiles/r02_small_call_pdl.txt
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/pdl_pytest.log 2>&1; echo "rc=$?" >> $OUT/pdl_pytest.log; tail -2 $OUT/pdl_pytest.log
python __graft_entry__.py smoke 2>&1 | tail -1
for r in 1 2; do
  HAMMING_LIB=tune_libs/nopdl.so python tools/c1_probe.py nopdl
  python tools/c1_probe.py pdl
done
