V='[{"tile_sizes":[4,1,1],"thread_shape":[128,1,1]},{"tile_sizes":[8,1,1],"thread_shape":[128,1,1]},{"tile_sizes":[8,1,1],"thread_shape":[256,1,1]},{"tile_sizes":[16,1,1],"thread_shape":[128,1,1]},{"tile_sizes":[16,1,1],"thread_shape":[512,1,1]},{"tile_sizes":[32,1,1],"thread_shape":[512,1,1]},{"tile_sizes":[4,1,1],"thread_shape":[64,1,1]}]'
timeout 200 python profiles/sweep.py kru "$V"
