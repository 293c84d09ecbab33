#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench, ncu launch list of the
# step and ncu --set full captures. Outputs under gpurun_out/$TAG.
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
rm -f gpurun_out/tc_errors.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
cp gpurun_out/tc_errors.jsonl $OUT/ 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_nt|fc_cluster|tc_gemm" -c 300 --csv \
    --log-file $OUT/launches.csv python bench.py --profile-only --steps 40 --warmup 3 > $OUT/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_nt|fc_cluster" -s 2 -c 6 \
    -o $OUT/step python profiles/ncu_ops.py tbmm 2fcrelu mlp3 > $OUT/ncu_step.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_nt|gconv|kru|lut" -c 4 \
    -o $OUT/ops python profiles/ncu_ops.py reps=1 c3 gconv kru lut > $OUT/ncu_ops.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm" -c 3 \
    -o $OUT/tc python profiles/ncu_ops.py math=tf32 reps=1 c3 tmm_huge > $OUT/ncu_tc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gconv" -c 2 \
    -o $OUT/tcgconv python profiles/ncu_ops.py math=tf32 reps=1 gconv > $OUT/ncu_tcgconv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_kru" -c 1 \
    -o $OUT/tckru python profiles/ncu_ops.py math=tf32 reps=1 kru > $OUT/ncu_tckru.log 2>&1
ls -la $OUT
