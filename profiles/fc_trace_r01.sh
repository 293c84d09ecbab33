# FC phase trace (profiles/fc_trace.cu) at the bench step's default plans
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_FC_TRACE -I paper_1802_04730_b200/csrc profiles/fc_trace.cu -o /tmp/fc_trace && /tmp/fc_trace
