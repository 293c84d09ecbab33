#!/bin/bash
OUT=gpurun_out/r02_gconv; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py -q -k "gconv" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for m in tf32 3xtf32; do timeout 300 python profiles/sweep.py gconv '[]' $m; done > $OUT/sweep.txt 2>&1
for op in gconv14 gconv7 gconv28 gconv56; do timeout 300 python profiles/sweep.py $op '[]' tf32; done >> $OUT/sweep.txt 2>&1
cat $OUT/sweep.txt; grep -E "passed|failed|Error" $OUT/pytest.log | tail -5
