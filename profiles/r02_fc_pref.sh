#!/bin/bash
# r02: FC parameter-line prefetch at entry: traces, timings, step
OUT=gpurun_out/r02_fc_pref; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_FC_TRACE -I paper_1802_04730_b200/csrc profiles/fc_trace.cu \
  paper_1802_04730_b200/csrc/kernels/attr.cu paper_1802_04730_b200/csrc/kernels/fc_tma.cu -o /tmp/fc_trace 2>&1 | grep -i error
/tmp/fc_trace > $OUT/trace.txt 2>&1; grep -A 26 "MLP3 rows=4 cn=4\]" $OUT/trace.txt; grep -A 22 "2FCRelu rows=4 cn=8\]" $OUT/trace.txt
for op in 2fcrelu mlp1 mlp3; do timeout 300 python profiles/sweep.py $op '[{}]' 2>&1 | tail -2; done > $OUT/sweep.txt 2>&1; cat $OUT/sweep.txt
COMBOS_ONLY=1 COMBOS_JSON='[{}, {}, {}]' timeout 600 python profiles/step_variants.py > $OUT/step.txt 2>&1; cat $OUT/step.txt | cut -c1-60
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fc_chain or golden" 2>&1 | tail -1
