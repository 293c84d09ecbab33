#!/bin/bash
# r02: 3xTF32 split with hi = the raw fp32 operand (rz), lo written once: TC parity + timings
OUT=gpurun_out/r02_x3; mkdir -p $OUT
rm -f gpurun_out/tc_errors.jsonl
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x > $OUT/pytest_tc.log 2>&1; echo "exit $?" >> $OUT/pytest_tc.log
tail -3 $OUT/pytest_tc.log
cp gpurun_out/tc_errors.jsonl $OUT/ 2>/dev/null
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -2 $OUT/smoke.log
for op in tmm_huge tmm_big c3 mlp3 2fcrelu tbmm; do
  timeout 300 python profiles/sweep.py $op '[]' 3xtf32 >> $OUT/sweep.txt 2>&1
  timeout 300 python profiles/sweep.py $op '[]' tf32 >> $OUT/sweep.txt 2>&1
done
cat $OUT/sweep.txt
