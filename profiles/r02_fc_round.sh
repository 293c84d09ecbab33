#!/bin/bash
# r02: FC chains — parity of the register chains, MLP3 plans, the step
OUT=gpurun_out/r02_fc; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "golden or fc_" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 300 python profiles/sweep.py mlp3 '[{"tile_sizes":[4,4,1],"thread_shape":[64,1,1],"fusion_strategy":"max"},{"tile_sizes":[1,1,2]},{"tile_sizes":[2,1,2]},{"tile_sizes":[4,1,2]}]' > $OUT/sweep_mlp3.txt 2>&1
timeout 300 python profiles/sweep.py 2fcrelu '[]' > $OUT/sweep_2fcrelu.txt 2>&1
COMBOS_ONLY=1 timeout 300 python profiles/step_variants.py > $OUT/step.txt 2>&1
cat $OUT/sweep_mlp3.txt $OUT/sweep_2fcrelu.txt; head -3 $OUT/step.txt; tail -2 $OUT/pytest.log
