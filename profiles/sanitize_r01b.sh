export PYTHONFAULTHANDLER=1
timeout 1800 compute-sanitizer --tool memcheck --print-limit 4 python -m pytest tests/test_gpu_parity.py -q -k "not paper_shape and not tuner" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|at .*\.cu" | head -20
timeout 1800 compute-sanitizer --tool memcheck --print-limit 4 python -m pytest tests/test_gpu_tc.py -q -k "not paper_shape and not 1024 and not 16384 and not tuner and not 500" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|at .*\.cu|not supported" | head -20
