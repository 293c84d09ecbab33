#!/bin/bash
# r02: producer-warp slab TBMM (one warp issues the copies, chunks on mbarriers): parity, trace, timings, step
OUT=gpurun_out/r02_slab_ws; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "every_gemm_variant or slab or golden" > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_SLAB_TRACE -I paper_1802_04730_b200/csrc profiles/slab_trace.cu \
  paper_1802_04730_b200/csrc/kernels/attr.cu paper_1802_04730_b200/csrc/kernels/gemm_tma.cu paper_1802_04730_b200/csrc/kernels/gemm_chunk.cu -o /tmp/slab_trace 2>&1 | grep -i "error" | head -5
for v in 54 53 57; do /tmp/slab_trace $v; done > $OUT/trace.txt 2>&1; cat $OUT/trace.txt
timeout 300 python profiles/sweep.py tbmm '[{"unroll_copy_shared":true},{"tile_sizes":[7,1,2],"unroll_copy_shared":true},{"tile_sizes":[5,1,2],"unroll_copy_shared":true},{"tile_sizes":[4,1,2],"unroll_copy_shared":true},{}]' > $OUT/sweep.txt 2>&1; cat $OUT/sweep.txt
COMBOS_ONLY=1 COMBOS_JSON='[{}, {"tbmm": {"unroll_copy_shared": true}}, {"tbmm": {"tile_sizes": [7, 1, 2], "unroll_copy_shared": true}}, {}, {"tbmm": {"unroll_copy_shared": true}}]' timeout 600 python profiles/step_variants.py > $OUT/step.txt 2>&1; cut -c1-200 $OUT/step.txt
