# compute-sanitizer memcheck + racecheck over the GPU parity tests (golden cases, small shapes)
export PYTHONFAULTHANDLER=1
K='golden and (small or ragged or zero)'
timeout 1200 compute-sanitizer --tool memcheck --print-limit 6 python -m pytest tests/test_gpu_parity.py -q -k "$K" 2>&1 | grep -v "^\s*$" | grep -E "passed|failed|ERROR SUMMARY|Invalid|at .*\.cu|Cluster" | head -30
timeout 1200 compute-sanitizer --tool racecheck --print-limit 6 python -m pytest tests/test_gpu_parity.py -q -k "$K" 2>&1 | grep -E "passed|failed|RACECHECK SUMMARY|hazard" | head -10
timeout 1200 compute-sanitizer --tool synccheck --print-limit 6 python -m pytest tests/test_gpu_parity.py -q -k "$K" 2>&1 | grep -E "passed|failed|ERROR SUMMARY" | head -10
