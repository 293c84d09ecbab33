#!/bin/bash
# r02: chunked warp-per-batch TBMM (gemm_chunk.cu): parity, phase traces, sweep
OUT=gpurun_out/r02_wchunk; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "wchunk or tbmm" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_WCHUNK_TRACE -I paper_1802_04730_b200/csrc \
  profiles/wchunk_trace.cu paper_1802_04730_b200/csrc/kernels/attr.cu -o /tmp/wchunk_trace 2>/dev/null
for cfg in "0 2 4" "0 2 2" "0 2 6" "0 1 4" "0 4 4" "0 2 1" "1 2 4"; do timeout 60 /tmp/wchunk_trace $cfg; done > $OUT/trace.txt 2>&1
cat $OUT/trace.txt
V='[{"tile_sizes":[7,4,4],"block_shape":[2,4,1]},{"tile_sizes":[7,4,4],"block_shape":[2,2,1]},{"tile_sizes":[7,4,4],"block_shape":[2,6,1]},{"tile_sizes":[7,4,4],"block_shape":[1,4,1]},{"tile_sizes":[7,4,4],"block_shape":[4,4,1]},{"tile_sizes":[7,4,4],"block_shape":[2,3,1]},{"tile_sizes":[4,4,4],"block_shape":[2,4,1]},{"tile_sizes":[7,1,2]}]'
timeout 300 python profiles/sweep.py tbmm "$V" > $OUT/sweep.txt 2>&1
cat $OUT/sweep.txt
