#!/bin/bash
OUT=gpurun_out/r02_fc_trace2; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_FC_TRACE -I paper_1802_04730_b200/csrc profiles/fc_trace.cu \
  paper_1802_04730_b200/csrc/kernels/attr.cu paper_1802_04730_b200/csrc/kernels/fc_tma.cu -o /tmp/fc_trace 2>&1 | grep -i error
/tmp/fc_trace > $OUT/trace.txt 2>&1; grep -A 24 "MLP3 rows=4 cn=4" $OUT/trace.txt | head -26; grep -A 16 "2FCRelu rows" $OUT/trace.txt | head -18
