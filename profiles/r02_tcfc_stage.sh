#!/bin/bash
# r02: tcgen05 FC chain with the epilogue staged in shared memory (coalesced stores): parity + timings
OUT=gpurun_out/r02_tcfc_stage; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
for m in tf32 3xtf32; do for op in mlp3 2fcrelu mlp1; do timeout 300 python profiles/sweep.py $op '[]' $m 2>&1 | tail -1; done; done > $OUT/sweep.txt 2>&1; cat $OUT/sweep.txt
