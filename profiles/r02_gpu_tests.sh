#!/bin/bash
# r02: the full GPU suite + smoke; tensor-core error records under gpurun_out/r02_tests
OUT=gpurun_out/r02_tests; mkdir -p $OUT
rm -f gpurun_out/tc_errors.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
cp gpurun_out/tc_errors.jsonl $OUT/ 2>/dev/null
tail -3 $OUT/smoke.log; grep -E "FAILED|passed|failed|exit" $OUT/pytest_gpu.log | tail -30
