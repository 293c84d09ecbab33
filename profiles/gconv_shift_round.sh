# shifted-halo tcgen05 gconv: tolerance tests, then paper-shape timings vs
# the other TC variants and the FFMA kernel
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_tc.py -x -q -k "gconv" > gpurun_out/shift_tests.log 2>&1
tail -4 gpurun_out/shift_tests.log
V='[{"tile_sizes":[128,16,3],"thread_shape":[512,1,1]},{"tile_sizes":[128,16,1],"thread_shape":[512,1,1]}]'
(timeout 200 python profiles/sweep.py gconv "$V" tf32; timeout 200 python profiles/sweep.py gconv "$V" 3xtf32; timeout 200 python profiles/sweep.py gconv '[]') > gpurun_out/shift_sweep.log 2>&1
cat gpurun_out/shift_sweep.log
