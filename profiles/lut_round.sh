timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_prodmodel.py -q -x -k "lut or prod or golden" 2>&1 | tail -3
python profiles/sweep.py lut '[{"thread_shape":[64,1,1]},{"thread_shape":[128,1,1]},{"thread_shape":[512,1,1]},{"thread_shape":[1024,1,1]}]'
