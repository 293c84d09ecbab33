#!/bin/bash
# r02: ncu --set full of the step's three kernels (one launch each, cold caches)
OUT=gpurun_out/r02_ncu; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_nt|fc_cluster" -c 3 \
    -o $OUT/step python profiles/ncu_ops.py reps=1 tbmm 2fcrelu mlp3 > $OUT/ncu_step.log 2>&1
python profiles/ncu_summary.py $OUT/ncu_step.json $OUT/step.ncu-rep > $OUT/ncu_step.txt 2>&1
cat $OUT/ncu_step.txt
