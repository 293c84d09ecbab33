#!/bin/bash
# r02: ncu launch list of the bench step + --set full captures of the step's
# kernels (slab TBMM, 2FCRelu / MLP3 cluster chains) and the TMA-fed C3.
OUT=gpurun_out/r02_ncu; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_nt|fc_cluster|fc_regs" -c 300 --csv \
    --log-file $OUT/launches.csv python bench.py --profile-only --steps 40 --warmup 3 > $OUT/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_nt|fc_cluster" -s 3 -c 3 \
    -o $OUT/step python profiles/ncu_ops.py tbmm 2fcrelu mlp3 > $OUT/ncu_step.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_nt" -s 1 -c 1 \
    -o $OUT/c3 python profiles/ncu_ops.py reps=2 c3 > $OUT/ncu_c3.log 2>&1
python profiles/launch_share.py $OUT/launches.csv $OUT/launch_share.json > $OUT/launch_share.txt 2>&1
python profiles/ncu_summary.py $OUT/ncu_full.json $OUT/step.ncu-rep $OUT/c3.ncu-rep > $OUT/ncu_full.txt 2>&1
cat $OUT/launch_share.txt $OUT/ncu_full.txt; tail -3 $OUT/ncu_step.log $OUT/ncu_c3.log
