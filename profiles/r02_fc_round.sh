#!/bin/bash
# r02: FC chains — parity, MLP3 / 2FCRelu / MLP1 plans (load modes), the step
OUT=gpurun_out/r02_fc; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "golden or fc_" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 300 python profiles/sweep.py mlp3 '[{"tile_sizes":[4,4,3]},{"tile_sizes":[4,4,4]},{"tile_sizes":[2,4,4]},{"tile_sizes":[2,2,4]},{"tile_sizes":[4,2,4]},{"tile_sizes":[8,4,4]},{"tile_sizes":[1,1,2]}]' > $OUT/sweep_mlp3.txt 2>&1
timeout 300 python profiles/sweep.py 2fcrelu '[{"tile_sizes":[4,8,3]},{"tile_sizes":[8,8,4],"thread_shape":[128,1,1]},{"tile_sizes":[2,8,4]},{"tile_sizes":[4,16,4]},{"tile_sizes":[8,16,4]}]' > $OUT/sweep_2fcrelu.txt 2>&1
timeout 300 python profiles/sweep.py mlp1 '[{"tile_sizes":[4,8,3]},{"tile_sizes":[4,8,4]},{"tile_sizes":[2,8,4]}]' > $OUT/sweep_mlp1.txt 2>&1
COMBOS_ONLY=1 timeout 300 python profiles/step_variants.py > $OUT/step.txt 2>&1
cat $OUT/sweep_mlp3.txt $OUT/sweep_2fcrelu.txt $OUT/sweep_mlp1.txt; cat $OUT/step.txt; tail -2 $OUT/pytest.log
