#!/bin/bash
# r02: persistent slab ring for TBMM (producer warp lands batch j+1 while batch j computes): parity, timings, step
OUT=gpurun_out/r02_slab_ring; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "slab_ring or slab_variants or golden" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
timeout 300 python profiles/sweep.py tbmm '[{"unroll_copy_shared":true,"block_shape":[1,1,2]},{"unroll_copy_shared":true,"block_shape":[1,1,3]},{"unroll_copy_shared":true,"block_shape":[1,2,2]},{"unroll_copy_shared":true,"block_shape":[1,2,3]},{"unroll_copy_shared":true,"block_shape":[1,3,2]},{"tile_sizes":[7,1,2],"unroll_copy_shared":true,"block_shape":[1,2,2]},{"tile_sizes":[5,1,2],"unroll_copy_shared":true,"block_shape":[1,2,3]},{}]' > $OUT/sweep.txt 2>&1; cat $OUT/sweep.txt
