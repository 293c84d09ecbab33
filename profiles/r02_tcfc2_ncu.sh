#!/bin/bash
OUT=gpurun_out/r02_tcfc2_ncu; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm" -s 2 -c 1 -o $OUT/fc2 python profiles/ncu_ops.py reps=3 math=tf32 2fcrelu > $OUT/ncu.log 2>&1
tail -n 2 $OUT/ncu.log
