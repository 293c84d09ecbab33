#!/bin/bash
OUT=gpurun_out/r02_x3_ncu; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm" -s 1 -c 1 -o $OUT/huge_x3 python profiles/ncu_ops.py math=3xtf32 tmm_huge > $OUT/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm" -s 1 -c 1 -o $OUT/huge_tf32 python profiles/ncu_ops.py math=tf32 tmm_huge > $OUT/ncu2.log 2>&1
tail -n 2 $OUT/ncu1.log; tail -n 2 $OUT/ncu2.log
