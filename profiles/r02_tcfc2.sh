#!/bin/bash
# r02: fused two-layer tcgen05 FC kernel (2FCRelu): TC parity + timings vs the per-layer launches
OUT=gpurun_out/r02_tcfc2; mkdir -p $OUT
rm -f gpurun_out/tc_errors.jsonl
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > $OUT/pytest_tc.log 2>&1; echo "exit $?" >> $OUT/pytest_tc.log
tail -3 $OUT/pytest_tc.log; cp gpurun_out/tc_errors.jsonl $OUT/ 2>/dev/null
for m in tf32 3xtf32; do
  timeout 300 python profiles/sweep.py 2fcrelu '[{"tile_sizes":[128,1,1],"fusion_strategy":"min"}]' $m 2>&1 | tail -2
done > $OUT/sweep.txt
cat $OUT/sweep.txt
