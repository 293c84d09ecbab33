#!/bin/bash
OUT=gpurun_out/r02_slab_l1; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "slab_variants or tbmm" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
V='[{"tile_sizes":[7,1,2],"unroll_copy_shared":true},{"tile_sizes":[4,1,2],"unroll_copy_shared":true},{"tile_sizes":[4,1,2]}]'
timeout 300 python profiles/sweep.py tbmm "$V" 2>&1 | tail -4
