#!/bin/bash
# r02: two-batch slab TBMM (a half-warp per batch, two columns per lane): parity, timings, step
OUT=gpurun_out/r02_slab2; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "slab2 or slab_variants or golden" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
timeout 300 python profiles/sweep.py tbmm '[{"block_shape":[1,2,1]},{"tile_sizes":[7,1,2],"block_shape":[1,2,1]},{"tile_sizes":[5,1,2],"block_shape":[1,2,1]},{}]' > $OUT/sweep.txt 2>&1; cat $OUT/sweep.txt
COMBOS_ONLY=1 COMBOS_JSON='[{}, {"tbmm": {"block_shape": [1, 2, 1]}}, {"tbmm": {"tile_sizes": [7, 1, 2], "block_shape": [1, 2, 1]}}, {}, {"tbmm": {"block_shape": [1, 2, 1]}}]' timeout 600 python profiles/step_variants.py > $OUT/step.txt 2>&1; cut -c1-120 $OUT/step.txt; grep -o '"step_us": [0-9.]*' $OUT/step.txt
