#!/bin/bash
# r02: bench N=1 (short), N=2 ranks sharing the one GPU (strong-split code path), GPU tests
OUT=gpurun_out/r02_bench; mkdir -p $OUT
timeout 900 python bench.py --steps 200 --warmup 10 > $OUT/bench1.json 2> $OUT/bench1.err; echo "bench1 exit $?" >> $OUT/bench1.err
timeout 600 python bench.py --gpus 2 --allow-shared-gpu --steps 100 --warmup 10 --no-ops > $OUT/bench2.json 2> $OUT/bench2.err; echo "bench2 exit $?" >> $OUT/bench2.err
timeout 120 python bench.py --gpus 2 --steps 10 > $OUT/bench2_strict.json 2> $OUT/bench2_strict.err; echo "strict exit $?" >> $OUT/bench2_strict.err
timeout 1500 python -m pytest tests/test_gpu_sharding.py tests/test_gpu_tc.py tests/test_gpu_parity.py -q > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
tail -2 $OUT/bench1.err $OUT/bench2.err $OUT/bench2_strict.err; grep -E "FAILED|passed|failed|exit" $OUT/pytest.log | tail
