#!/bin/bash
OUT=gpurun_out/r02_e2e; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sliced or host_buffers" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for n in 1 2 3 4 6; do TCB_HOST_SLICES=$n timeout 300 python profiles/e2e_slices.py; done > $OUT/slices.txt 2>&1
cat $OUT/slices.txt
