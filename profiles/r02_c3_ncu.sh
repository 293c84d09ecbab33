#!/bin/bash
OUT=gpurun_out/r02_c3_ncu; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_nt" -s 2 -c 1 -o $OUT/c3 python profiles/ncu_ops.py reps=3 c3 > $OUT/ncu.log 2>&1
tail -n 1 $OUT/ncu.log
