# tcgen05 3-KRU: tolerance tests, then paper-shape timings vs the FFMA kernel
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "kru or refuses or unsupported or mapping" > gpurun_out/kru_tests.log 2>&1
tail -15 gpurun_out/kru_tests.log
(timeout 100 python profiles/sweep.py kru '[]' tf32; timeout 100 python profiles/sweep.py kru '[]' 3xtf32; timeout 100 python profiles/sweep.py kru '[]') 2>&1 | tail -3
