#!/bin/bash
OUT=gpurun_out/r02_fc_sweep; mkdir -p $OUT
V3='[{"tile_sizes":[8,4,1],"thread_shape":[128,1,1]},{"tile_sizes":[8,2,1],"thread_shape":[256,1,1]},{"tile_sizes":[16,4,1],"thread_shape":[256,1,1]},{"tile_sizes":[8,8,1],"thread_shape":[64,1,1]},{"tile_sizes":[16,8,1],"thread_shape":[128,1,1]},{"tile_sizes":[8,1,1],"thread_shape":[512,1,1]},{"tile_sizes":[16,2,1],"thread_shape":[512,1,1]}]'
timeout 300 python profiles/sweep.py mlp3 "$V3" > $OUT/mlp3.txt 2>&1
V2='[{"tile_sizes":[8,8,1],"thread_shape":[128,1,1]},{"tile_sizes":[8,16,1],"thread_shape":[64,1,1]},{"tile_sizes":[16,16,1],"thread_shape":[128,1,1]},{"tile_sizes":[8,4,1],"thread_shape":[256,1,1]},{"tile_sizes":[16,8,1],"thread_shape":[256,1,1]}]'
timeout 300 python profiles/sweep.py 2fcrelu "$V2" > $OUT/2fcrelu.txt 2>&1
cat $OUT/mlp3.txt $OUT/2fcrelu.txt
