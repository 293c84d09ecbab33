#!/bin/bash
# r02 fourth pass (FC copies issued first): ncu --set full of the step kernels at their defaults, the bench's launch list,
# then the driver's round-end sequence (GPU tests, smoke, reference arm, bench with driver args)
OUT=gpurun_out/r02_final6; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_nt|fc_cluster" -c 3 \
    -o $OUT/step python profiles/ncu_ops.py reps=1 tbmm 2fcrelu mlp3 > $OUT/ncu_step.log 2>&1
python profiles/ncu_summary.py $OUT/ncu_step.json $OUT/step.ncu-rep > $OUT/ncu_step.txt 2>&1
cat $OUT/ncu_step.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_nt|fc_|copy|tc_" -c 600 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 > $OUT/bench_under_ncu.log 2>&1
echo "launches exit $?"
rm -f gpurun_out/tc_errors.jsonl
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
cp gpurun_out/tc_errors.jsonl $OUT/ 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
tail -2 $OUT/pytest_gpu.log; tail -3 $OUT/smoke.log; tail -1 $OUT/bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02_final6/bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"]["us_per_step"], "clocks", d["clocks"]["sm_mhz"], d["clocks"]["window"]["samples"])
r = d["roofline"]; print("roofline", r["kernel"], r["frac"], r["traffic"])
for k, v in r["by_kernel"].items(): print("  ", k, v)
print("prod", d["prod_model"].get("us_per_forward"))
ref = json.loads(open("gpurun_out/r02_final6/bench_ref.json").read().strip().splitlines()[-1])
print("ref", ref["value"], ref["config"] == d["config"])
PY
