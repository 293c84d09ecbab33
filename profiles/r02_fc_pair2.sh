#!/bin/bash
# r02: column-pair FC chains with 16-step chunks: parity + timings
OUT=gpurun_out/r02_fc_pair2; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fc_chain_cluster" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_FC_TRACE -I paper_1802_04730_b200/csrc profiles/fc_trace.cu \
  paper_1802_04730_b200/csrc/kernels/attr.cu paper_1802_04730_b200/csrc/kernels/fc_tma.cu -o /tmp/fc_trace 2>&1 | grep -i error
FC_TRACE_2FC=1 FC_TRACE_PAIR_ONLY=1 /tmp/fc_trace > $OUT/trace.txt 2>&1
grep "no error\|L0_enter\|L0_chain" $OUT/trace.txt
for op in 2fcrelu mlp1; do
  timeout 300 python profiles/sweep.py $op '[{"thread_shape":[32,1,1]},{"tile_sizes":[8,8,1],"thread_shape":[64,1,1]},{"tile_sizes":[2,8,1],"thread_shape":[32,1,1]}]' 2>&1 | tail -4
done > $OUT/sweep.txt 2>&1
cat $OUT/sweep.txt
