#!/bin/bash
# r02: FC chains with layer 0 streamed by TMA chunks (fc_tma.cu, tile_sizes[2] == 6): parity + sweeps
OUT=gpurun_out/r02_fctma; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fc_tma or fc_chain or golden" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
V2='[{"tile_sizes":[4,8,6],"thread_shape":[64,1,1]},{"tile_sizes":[8,8,6],"thread_shape":[128,1,1]},{"tile_sizes":[8,8,6],"thread_shape":[64,1,1]},{"tile_sizes":[16,8,6],"thread_shape":[256,1,1]},{"tile_sizes":[8,16,6],"thread_shape":[64,1,1]},{"tile_sizes":[4,16,6],"thread_shape":[32,1,1]},{"tile_sizes":[8,4,6],"thread_shape":[256,1,1]},{"tile_sizes":[8,8,1],"thread_shape":[128,1,1]}]'
timeout 300 python profiles/sweep.py 2fcrelu "$V2" > $OUT/sweep_2fcrelu.txt 2>&1
timeout 300 python profiles/sweep.py mlp1 "$V2" > $OUT/sweep_mlp1.txt 2>&1
timeout 300 python profiles/sweep.py mlp3 '[{"tile_sizes":[4,4,6],"thread_shape":[64,1,1]},{"tile_sizes":[8,4,6],"thread_shape":[128,1,1]},{"tile_sizes":[8,8,6],"thread_shape":[64,1,1]}]' > $OUT/sweep_mlp3.txt 2>&1
cat $OUT/sweep_2fcrelu.txt $OUT/sweep_mlp1.txt $OUT/sweep_mlp3.txt
