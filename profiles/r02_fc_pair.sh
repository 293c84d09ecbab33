#!/bin/bash
# r02: column-pair FC chains (two outputs per lane): phase traces + library timings
OUT=gpurun_out/r02_fc_pair; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_FC_TRACE -I paper_1802_04730_b200/csrc profiles/fc_trace.cu \
  paper_1802_04730_b200/csrc/kernels/attr.cu paper_1802_04730_b200/csrc/kernels/fc_tma.cu -o /tmp/fc_trace 2>&1 | grep -i error
FC_TRACE_2FC=1 FC_TRACE_PAIR_ONLY=1 /tmp/fc_trace > $OUT/trace.txt 2>&1; cat $OUT/trace.txt | grep -v "^  [a-z]" 
grep -A 30 "column pairs" $OUT/trace.txt | grep "L0_enter\|L0_chain\|L1_enter\|L1_chain\|end " 
for op in 2fcrelu mlp1 mlp3; do
  timeout 300 python profiles/sweep.py $op '[{"thread_shape":[32,1,1]},{"tile_sizes":[8,8,1],"thread_shape":[64,1,1]},{"tile_sizes":[4,4,1],"thread_shape":[32,1,1]},{"tile_sizes":[8,4,1],"thread_shape":[64,1,1]}]' 2>&1 | tail -5
done > $OUT/sweep.txt 2>&1
cat $OUT/sweep.txt
