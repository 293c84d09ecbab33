#!/bin/bash
OUT=gpurun_out/r02_check; mkdir -p $OUT
timeout 300 python profiles/sweep.py tmm_huge '[{"tile_sizes":[32,32,64],"thread_shape":[16,16,1],"block_shape":[1,1,1]},{"tile_sizes":[32,32,3],"thread_shape":[16,8,1],"block_shape":[1,1,1]}]' > $OUT/sweep_huge.txt 2>&1
timeout 900 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
cat $OUT/sweep_huge.txt; python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02_check/bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"]["us_per_step"])
print("roofline", d["roofline"]["kernel"], d["roofline"]["frac"])
for k, v in d["step_ops"].items(): print(" ", k, v["us"], v["kernel"])
for k, v in d["ops"].items():
    print("%-40s %9s %s %s" % (k, v.get("us"), v.get("kernel", v.get("error")), (v.get("capi_sync_latency") or {}).get("us_p0_p50_p90_p99")))
print("prod", d["prod_model"].get("us_per_forward"), d["prod_model"].get("kernels"))
PY
