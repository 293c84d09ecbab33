#!/bin/bash
# r02: the driver's round-end sequence on one box: GPU tests, smoke, reference arm, bench (driver args)
OUT=gpurun_out/r02_final; mkdir -p $OUT
rm -f gpurun_out/tc_errors.jsonl
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
cp gpurun_out/tc_errors.jsonl $OUT/ 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
tail -2 $OUT/pytest_gpu.log; tail -3 $OUT/smoke.log; tail -1 $OUT/bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02_final/bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"]["us_per_step"], "clocks", d["clocks"])
r = d["roofline"]; print("roofline", r["kernel"], r["frac"], r["traffic"], r["chain_floor_frac"])
for k, v in r["by_kernel"].items(): print("  ", k, v)
print("cpu", d.get("cpu_baseline", {}).get("value"), d.get("cpu_baseline_port", {}).get("value"))
print("prod", d["prod_model"].get("us_per_forward"))
ref = json.loads(open("gpurun_out/r02_final/bench_ref.json").read().strip().splitlines()[-1])
print("ref", ref["value"], ref["config"] == d["config"])
PY
