#!/bin/bash
# r02: phase trace of the default TBMM kernel (slab_c9, variant 53) and slab_c4/c7, cold operands
OUT=gpurun_out/r02_slab_trace9; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_SLAB_TRACE -I paper_1802_04730_b200/csrc profiles/slab_trace.cu \
  paper_1802_04730_b200/csrc/kernels/attr.cu paper_1802_04730_b200/csrc/kernels/gemm_tma.cu paper_1802_04730_b200/csrc/kernels/gemm_chunk.cu -o /tmp/slab_trace 2>&1 | grep -i "error" | head -5
for v in 53 29 30; do /tmp/slab_trace $v; done > $OUT/trace.txt 2>&1; cat $OUT/trace.txt
