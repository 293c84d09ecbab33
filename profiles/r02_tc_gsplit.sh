#!/bin/bash
# r02: global split-K (no cluster) for 96/112-wide tcgen05 tiles: the huge TMM on all 148 SMs
OUT=gpurun_out/r02_tc_gsplit; mkdir -p $OUT
rm -f gpurun_out/tc_errors.jsonl
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > $OUT/pytest_tc.log 2>&1; tail -2 $OUT/pytest_tc.log; cp gpurun_out/tc_errors.jsonl $OUT/
for m in tf32 3xtf32; do
  timeout 300 python profiles/sweep.py tmm_huge '[{"tile_sizes":[128,128,32],"block_shape":[1,1,4]},{"tile_sizes":[128,112,32],"block_shape":[1,1,4]},{"tile_sizes":[128,96,32],"block_shape":[1,1,4]},{"tile_sizes":[128,112,32],"block_shape":[1,1,8]}]' $m 2>&1 | tail -5
done > $OUT/sweep.txt 2>&1; cat $OUT/sweep.txt
