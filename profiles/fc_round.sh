timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fc or golden or mlp" 2>&1 | tail -3
bash profiles/fc_trace_r01.sh 2>&1 | grep -E "^[A-Z0-9]|L[0-9]_|copies|globaltimer" | head -60
python profiles/sweep.py mlp3 '[{"tile_sizes":[4,4,1],"thread_shape":[64,1,1]},{"tile_sizes":[8,4,1],"thread_shape":[128,1,1]},{"tile_sizes":[2,2,1],"thread_shape":[64,1,1]},{"tile_sizes":[4,2,1],"thread_shape":[128,1,1]},{"tile_sizes":[8,2,1],"thread_shape":[256,1,1]}]'
python profiles/sweep.py 2fcrelu '[{"tile_sizes":[2,8,1],"thread_shape":[64,1,1]},{"tile_sizes":[8,8,1],"thread_shape":[128,1,1]},{"tile_sizes":[4,16,1],"thread_shape":[64,1,1]},{"tile_sizes":[8,16,1],"thread_shape":[64,1,1]}]'
