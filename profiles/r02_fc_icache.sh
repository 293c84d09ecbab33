#!/bin/bash
# r02: FC cluster kernel with the load mode as a template parameter and the chain as a shared
# (non-inlined) function: smaller instruction footprint. Parity, per-op sweep, trace, step.
OUT=gpurun_out/r02_fc_icache; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fc or mlp or golden or 2fcrelu" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for op in mlp3 2fcrelu mlp1; do timeout 300 python profiles/sweep.py $op '[]' 2>&1 | tail -1; done > $OUT/sweep.txt
cat $OUT/sweep.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_FC_TRACE -I paper_1802_04730_b200/csrc profiles/fc_trace.cu \
  paper_1802_04730_b200/csrc/kernels/attr.cu paper_1802_04730_b200/csrc/kernels/fc_tma.cu -o /tmp/fc_trace 2>&1 | grep -i error
/tmp/fc_trace > $OUT/trace.txt 2>&1; grep -A 20 "MLP3 rows=4 cn=4" $OUT/trace.txt | head -20
ORDER_ONLY=1 timeout 300 python profiles/step_variants.py 2>&1 | head -2
