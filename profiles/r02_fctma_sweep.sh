OUT=gpurun_out/fctma; mkdir -p $OUT
V2='[{"tile_sizes":[4,8,6],"thread_shape":[64,1,1]},{"tile_sizes":[8,8,6],"thread_shape":[128,1,1]},{"tile_sizes":[8,8,6],"thread_shape":[64,1,1]},{"tile_sizes":[16,8,6],"thread_shape":[256,1,1]},{"tile_sizes":[8,16,6],"thread_shape":[64,1,1]},{"tile_sizes":[4,16,6],"thread_shape":[64,1,1]},{"tile_sizes":[8,4,6],"thread_shape":[256,1,1]},{"tile_sizes":[4,8,1],"thread_shape":[64,1,1]}]'
timeout 300 python profiles/sweep.py 2fcrelu "$V2" > $OUT/sweep_2fcrelu.txt 2>&1
timeout 300 python profiles/sweep.py mlp3 '[{"tile_sizes":[4,4,6],"thread_shape":[64,1,1]},{"tile_sizes":[8,4,6],"thread_shape":[128,1,1]},{"tile_sizes":[8,8,6],"thread_shape":[64,1,1]},{"tile_sizes":[4,8,6],"thread_shape":[64,1,1]}]' > $OUT/sweep_mlp3.txt 2>&1
cat $OUT/sweep_2fcrelu.txt $OUT/sweep_mlp3.txt
