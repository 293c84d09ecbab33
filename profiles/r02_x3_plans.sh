#!/bin/bash
# r02: 3xTF32 (rz hi) parity + plan sweep for the huge TMM and C3
OUT=gpurun_out/r02_x3plans; mkdir -p $OUT
rm -f gpurun_out/tc_errors.jsonl
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > $OUT/pytest_tc.log 2>&1; echo "exit $?" >> $OUT/pytest_tc.log
tail -2 $OUT/pytest_tc.log; cp gpurun_out/tc_errors.jsonl $OUT/ 2>/dev/null
V='[{"tile_sizes":[128,128,1],"block_shape":[1,1,1]},{"tile_sizes":[128,128,1],"block_shape":[1,1,2]},{"tile_sizes":[128,128,1],"block_shape":[1,1,4]},{"tile_sizes":[128,128,1],"block_shape":[1,1,8]},{"tile_sizes":[128,256,1],"block_shape":[1,1,2]},{"tile_sizes":[128,256,1],"block_shape":[1,1,4]},{"tile_sizes":[128,256,1],"block_shape":[1,1,8]},{"tile_sizes":[128,64,1],"block_shape":[1,1,2]}]'
for op in tmm_huge c3; do timeout 400 python profiles/sweep.py $op "$V" 3xtf32 >> $OUT/sweep.txt 2>&1; done
cat $OUT/sweep.txt
