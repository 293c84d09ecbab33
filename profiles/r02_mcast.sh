#!/bin/bash
# r02: tcgen05 GEMM with the A k-block multicast over N-tile pairs: parity + timings (on / off)
OUT=gpurun_out/r02_mcast; mkdir -p $OUT
rm -f gpurun_out/tc_errors.jsonl
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > $OUT/pytest_tc.log 2>&1; echo "exit $?" >> $OUT/pytest_tc.log
tail -2 $OUT/pytest_tc.log; cp gpurun_out/tc_errors.jsonl $OUT/ 2>/dev/null
for mc in 1 0; do
  for op in tmm_huge tmm_big c3; do
    for m in tf32 3xtf32; do echo "mcast=$mc $op $m: $(TCB_TC_MCAST=$mc timeout 300 python profiles/sweep.py $op '[]' $m 2>&1 | tail -1)"; done
  done
done > $OUT/sweep.txt
cat $OUT/sweep.txt
