#!/bin/bash
# r02: 3xTF32 tcgen05 GEMM with B's lo half written over the landed A (6-deep ring at BN=128)
OUT=gpurun_out/r02_x3_loina; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
for op in tmm_huge tmm_big c3; do timeout 300 python profiles/sweep.py $op '[]' 3xtf32 2>&1 | tail -1; done > $OUT/sweep.txt 2>&1
for op in tmm_huge c3; do timeout 300 python profiles/sweep.py $op '[]' tf32 2>&1 | tail -1; done >> $OUT/sweep.txt 2>&1; cat $OUT/sweep.txt
