#!/bin/bash
OUT=gpurun_out/r02_wpair_ncu; mkdir -p $OUT
O='{"tile_sizes":[7,4,4],"block_shape":[2,1,1],"fusion_strategy":"max","rng_seed":0,"shared_memory_budget":49152,"thread_shape":[32,1,1],"unroll_copy_shared":false,"unroll_factor":1,"use_private":true,"use_shared":true}'
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_nt" -s 1 -c 1 -o $OUT/wpair python profiles/ncu_ops.py "opts=$O" tbmm > $OUT/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_nt" -s 1 -c 1 -o $OUT/slab python profiles/ncu_ops.py tbmm > $OUT/ncu2.log 2>&1
tail -2 $OUT/ncu1.log $OUT/ncu2.log
