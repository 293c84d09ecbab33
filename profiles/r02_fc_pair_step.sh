#!/bin/bash
# r02: column-pair 2FCRelu / MLP1 in the bench step and alone
OUT=gpurun_out/r02_fc_pair_step; mkdir -p $OUT
COMBOS_ONLY=1 COMBOS_JSON='[{"2FCRelu": {"thread_shape": [32, 1, 1]}}, {}, {"2FCRelu": {"thread_shape": [32, 1, 1]}}, {}, {"2FCRelu": {"thread_shape": [32, 1, 1]}, "tbmm": {"tile_sizes": [4, 1, 2]}}, {"tbmm": {"tile_sizes": [4, 1, 2]}}]' \
  timeout 600 python profiles/step_variants.py > $OUT/step.txt 2>&1; cat $OUT/step.txt
for op in 2fcrelu mlp1; do timeout 300 python profiles/sweep.py $op '[{"thread_shape":[32,1,1]},{},{"thread_shape":[32,1,1]}]' 2>&1 | tail -4; done > $OUT/sweep.txt 2>&1; cat $OUT/sweep.txt
