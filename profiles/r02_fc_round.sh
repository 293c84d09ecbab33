#!/bin/bash
# r02: FC chains — parity, 2x2 chain tiles vs single chains, the step
OUT=gpurun_out/r02_fc; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "golden or fc_" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 300 python profiles/sweep.py 2fcrelu '[{"tile_sizes":[4,8,6],"thread_shape":[32,1,1]},{"tile_sizes":[8,8,6],"thread_shape":[32,1,1]},{"tile_sizes":[8,8,6],"thread_shape":[64,1,1]},{"tile_sizes":[16,8,6],"thread_shape":[64,1,1]},{"tile_sizes":[8,4,6],"thread_shape":[64,1,1]},{"tile_sizes":[16,8,6],"thread_shape":[128,1,1]}]' > $OUT/sweep_2fcrelu.txt 2>&1
timeout 300 python profiles/sweep.py mlp3 '[{"tile_sizes":[4,4,6],"thread_shape":[32,1,1]},{"tile_sizes":[8,4,6],"thread_shape":[32,1,1]},{"tile_sizes":[8,4,6],"thread_shape":[64,1,1]},{"tile_sizes":[4,2,6],"thread_shape":[32,1,1]}]' > $OUT/sweep_mlp3.txt 2>&1
timeout 300 python profiles/sweep.py mlp1 '[{"tile_sizes":[8,8,6],"thread_shape":[32,1,1]},{"tile_sizes":[4,8,6],"thread_shape":[32,1,1]},{"tile_sizes":[16,8,6],"thread_shape":[64,1,1]}]' > $OUT/sweep_mlp1.txt 2>&1
cat $OUT/sweep_2fcrelu.txt $OUT/sweep_mlp3.txt $OUT/sweep_mlp1.txt; tail -3 $OUT/pytest.log
