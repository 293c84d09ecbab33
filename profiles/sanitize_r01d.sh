# compute-sanitizer on the tcgen05 3-KRU and the shifted-halo gconv (small cases)
export PYTHONFAULTHANDLER=1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 6 python -m pytest tests/test_gpu_tc.py -q -k "kru" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|at .*\.cu" | head -12
timeout 1500 compute-sanitizer --tool racecheck --print-limit 6 python -m pytest tests/test_gpu_tc.py -q -k "kru or (gconv_tc and shift and not paper)" 2>&1 | grep -E "passed|failed|RACECHECK SUMMARY|hazard" | head -10
timeout 1500 compute-sanitizer --tool synccheck --print-limit 6 python -m pytest tests/test_gpu_tc.py -q -k "kru or (gconv_tc and shift and not paper)" 2>&1 | grep -E "passed|failed|ERROR SUMMARY" | head -10
