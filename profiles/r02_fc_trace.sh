#!/bin/bash
OUT=gpurun_out/r02_fc_trace; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_FC_TRACE -I paper_1802_04730_b200/csrc profiles/fc_trace.cu \
  paper_1802_04730_b200/csrc/kernels/attr.cu paper_1802_04730_b200/csrc/kernels/fc_tma.cu -o /tmp/fc_trace 2>&1 | grep -i error
/tmp/fc_trace > $OUT/trace.txt 2>&1
V='[{"tile_sizes":[4,4,1],"thread_shape":[64,1,1]}]'
timeout 300 python profiles/sweep.py mlp3 "$V" > $OUT/sweep.txt 2>&1
timeout 300 python profiles/sweep.py 2fcrelu '[]' >> $OUT/sweep.txt 2>&1
cat $OUT/trace.txt $OUT/sweep.txt
