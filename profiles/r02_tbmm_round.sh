#!/bin/bash
# r02: slab TBMM kernel — parity + standalone time vs the r01 plans
OUT=gpurun_out/r02_tbmm; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or variant or batched" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 300 python profiles/sweep.py mlp3 '[{"tile_sizes":[4,4,1],"thread_shape":[64,1,1]},{"tile_sizes":[1,1,2]},{"tile_sizes":[2,1,2]},{"tile_sizes":[4,1,2]}]' > $OUT/sweep.txt 2>&1
COMBOS_ONLY=1 timeout 300 python profiles/step_variants.py > $OUT/step.txt 2>&1
cat $OUT/sweep.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_SLAB_TRACE -I paper_1802_04730_b200/csrc profiles/slab_trace.cu -o /tmp/slab_trace 2>/dev/null && for v in 35 37 38; do /tmp/slab_trace $v; done > gpurun_out/r02_tbmm/trace.txt
cat gpurun_out/r02_tbmm/trace.txt
