# e2e host-path round: pinned/host parity tests, the e2e probe (copy
# bandwidth, per-call cost, step variants), then a short bench
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "pinned or host" > gpurun_out/pin_tests.log 2>&1
tail -3 gpurun_out/pin_tests.log
timeout 300 python profiles/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
cat gpurun_out/e2e_probe.log
timeout 600 python bench.py --steps 400 --warmup 20 > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
python -c "import json;d=json.load(open('gpurun_out/bench_e2e.json'));print(d['value'],d['ms_per_step'],d['e2e'])"
