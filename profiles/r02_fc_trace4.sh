#!/bin/bash
# r02: phase traces of the default FC plans after the early-copy change
OUT=gpurun_out/r02_fc_trace4; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_FC_TRACE -I paper_1802_04730_b200/csrc profiles/fc_trace.cu \
  paper_1802_04730_b200/csrc/kernels/attr.cu paper_1802_04730_b200/csrc/kernels/fc_tma.cu -o /tmp/fc_trace 2>&1 | grep -i error
/tmp/fc_trace > $OUT/trace.txt 2>&1; grep -A 26 "MLP3 rows=4 cn=4\]" $OUT/trace.txt; grep -A 3 "MLP3 rows=1 cn=1\]" $OUT/trace.txt; grep -A 3 "MLP3 rows=2 cn=4\]" $OUT/trace.txt
for v in '[{"tile_sizes":[1,1,1],"thread_shape":[64,1,1]},{"tile_sizes":[2,1,1],"thread_shape":[128,1,1]},{"tile_sizes":[2,2,1],"thread_shape":[64,1,1]},{"tile_sizes":[4,2,1],"thread_shape":[64,1,1]},{"tile_sizes":[2,4,1],"thread_shape":[32,1,1]},{"tile_sizes":[8,4,1],"thread_shape":[128,1,1]},{"tile_sizes":[4,4,1],"thread_shape":[32,1,1]}]'; do
  timeout 300 python profiles/sweep.py mlp3 "$v" 2>&1 | tail -8; done > $OUT/sweep_mlp3.txt 2>&1; cat $OUT/sweep_mlp3.txt
