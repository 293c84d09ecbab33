#!/bin/bash
OUT=gpurun_out/r02_mlp3_ncu; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fc_cluster" -s 2 -c 1 -o $OUT/mlp3 python profiles/ncu_ops.py reps=3 mlp3 > $OUT/ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fc_cluster" -s 2 -c 1 -o $OUT/fc2 python profiles/ncu_ops.py reps=3 2fcrelu > $OUT/ncu2.log 2>&1
tail -n 1 $OUT/ncu.log
