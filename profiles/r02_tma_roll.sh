#!/bin/bash
OUT=gpurun_out/r02_tma_roll; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tma_gemm or golden" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for op in c3 tmm_big tmm_huge; do timeout 300 python profiles/sweep.py $op '[]' 2>&1 | tail -1; done
