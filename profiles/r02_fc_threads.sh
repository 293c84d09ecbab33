#!/bin/bash
OUT=gpurun_out/r02_fc_threads; mkdir -p $OUT
timeout 300 python profiles/sweep.py mlp3 '[{"thread_shape":[128,1,1]},{"thread_shape":[256,1,1]},{"tile_sizes":[8,4,1],"thread_shape":[256,1,1]}]' > $OUT/mlp3.txt 2>&1
timeout 300 python profiles/sweep.py 2fcrelu '[{"thread_shape":[128,1,1]},{"thread_shape":[256,1,1]}]' > $OUT/2fcrelu.txt 2>&1
cat $OUT/mlp3.txt $OUT/2fcrelu.txt
