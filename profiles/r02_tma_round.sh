#!/bin/bash
OUT=gpurun_out/r02_tma; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tma or golden" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
V='[{"tile_sizes":[32,32,3],"thread_shape":[16,16,1],"block_shape":[1,1,1]},{"tile_sizes":[32,32,3],"thread_shape":[16,8,1],"block_shape":[1,1,1]},{"tile_sizes":[16,32,3],"thread_shape":[8,8,1],"block_shape":[1,1,1]},{"tile_sizes":[32,16,3],"thread_shape":[8,8,1],"block_shape":[1,1,1]}]'
for op in c3 tmm_huge; do echo "== $op"; timeout 300 python profiles/sweep.py $op "$V"; done > $OUT/sweep.txt 2>&1
cat $OUT/sweep.txt; tail -3 $OUT/pytest.log
