# compute-sanitizer over the round's new device code: the shifted-halo tcgen05
# gconv (small and odd-plane cases), the FC chain templated on its layer count,
# and the host segment-copy kernel (pinned host tensors)
export PYTHONFAULTHANDLER=1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 6 python -m pytest tests/test_gpu_tc.py -q -k "gconv_tc and shift and not paper" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|at .*\.cu" | head -20
timeout 1500 compute-sanitizer --tool memcheck --print-limit 6 python -m pytest tests/test_gpu_parity.py -q -k "pinned or host or (golden and (fc or mlp or 2fcrelu) and small)" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|at .*\.cu" | head -20
timeout 1500 compute-sanitizer --tool racecheck --print-limit 6 python -m pytest tests/test_gpu_parity.py -q -k "golden and (mlp3 or 2fcrelu) and small" 2>&1 | grep -E "passed|failed|RACECHECK SUMMARY|hazard" | head -10
