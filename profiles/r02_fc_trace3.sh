#!/bin/bash
# r02: phase traces of other 2FCRelu cluster plans (why rows=8 cn=8 t=128 is 2x slower)
OUT=gpurun_out/r02_fc_trace3; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_FC_TRACE -I paper_1802_04730_b200/csrc profiles/fc_trace.cu \
  paper_1802_04730_b200/csrc/kernels/attr.cu paper_1802_04730_b200/csrc/kernels/fc_tma.cu -o /tmp/fc_trace 2>&1 | grep -i error
FC_TRACE_2FC=1 /tmp/fc_trace > $OUT/trace.txt 2>&1; cat $OUT/trace.txt
