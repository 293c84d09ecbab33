#!/bin/bash
# r02: 96/112-wide tcgen05 GEMM tiles so the huge TMM grid covers all 148 SMs (37 x 4 = 148 CTAs vs 32 x 4 = 128)
OUT=gpurun_out/r02_tc_bn112; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > $OUT/pytest_tc.log 2>&1; tail -2 $OUT/pytest_tc.log
for m in tf32 3xtf32; do
  timeout 300 python profiles/sweep.py tmm_huge '[{"tile_sizes":[128,128,32],"block_shape":[1,1,4]},{"tile_sizes":[128,112,32],"block_shape":[1,1,4]},{"tile_sizes":[128,96,32],"block_shape":[1,1,4]},{"tile_sizes":[128,112,32],"block_shape":[1,1,2]}]' $m 2>&1 | tail -5
  timeout 300 python profiles/sweep.py tmm_big '[{"tile_sizes":[128,128,32],"block_shape":[1,1,8]},{"tile_sizes":[128,64,32],"block_shape":[1,1,8]},{"tile_sizes":[128,112,32],"block_shape":[1,1,8]},{"tile_sizes":[128,64,32],"block_shape":[1,1,4]}]' $m 2>&1 | tail -5
done > $OUT/sweep.txt 2>&1; cat $OUT/sweep.txt
