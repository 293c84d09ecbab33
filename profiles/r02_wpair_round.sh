#!/bin/bash
# r02: FFMA2 warp-tile TBMM (gemm_chunk.cu): parity, phase traces, sweep
OUT=gpurun_out/r02_wpair; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "wpair or tbmm" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_WPAIR_TRACE -I paper_1802_04730_b200/csrc \
  profiles/wpair_trace.cu paper_1802_04730_b200/csrc/kernels/attr.cu -o /tmp/wpair_trace 2>/dev/null
for cfg in "0 2" "1 2" "1 4"; do timeout 60 /tmp/wpair_trace $cfg; TCB_WPAIR_STG=1 timeout 60 /tmp/wpair_trace $cfg; done > $OUT/trace.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_SLAB_TRACE -I paper_1802_04730_b200/csrc profiles/slab_trace.cu -o /tmp/slab_trace 2>/dev/null && for v in 29 30; do /tmp/slab_trace $v; done >> $OUT/trace.txt 2>&1
cat $OUT/trace.txt
V='[{"tile_sizes":[7,4,4],"block_shape":[1,1,1]},{"tile_sizes":[7,4,4],"block_shape":[2,1,1]},{"tile_sizes":[7,4,4],"block_shape":[4,1,1]},{"tile_sizes":[4,4,4],"block_shape":[2,1,1]},{"tile_sizes":[4,4,4],"block_shape":[4,1,1]},{"tile_sizes":[4,4,4],"block_shape":[8,1,1]},{"tile_sizes":[7,1,2]}]'
timeout 300 python profiles/sweep.py tbmm "$V" > $OUT/sweep.txt 2>&1
cat $OUT/sweep.txt
