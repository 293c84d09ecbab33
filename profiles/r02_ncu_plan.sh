#!/bin/bash
# r02: ncu --set full of the bench's TBMM plan (STEP_PLANS: slab, tile_sizes [4,1,2]) + the
# launch list of the bench command itself (per-launch times, cold, serialised)
OUT=gpurun_out/r02_ncu_plan; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_nt" -c 1 \
    -o $OUT/tbmm python profiles/ncu_ops.py reps=1 'opts={"tile_sizes":[4,1,2]}' tbmm > $OUT/ncu_tbmm.log 2>&1
python profiles/ncu_summary.py $OUT/ncu_tbmm.json $OUT/tbmm.ncu-rep > $OUT/ncu_tbmm.txt 2>&1
cat $OUT/ncu_tbmm.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_nt|fc_|copy|tc_" -c 600 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 > $OUT/bench_under_ncu.log 2>&1
echo "launches exit $?"
