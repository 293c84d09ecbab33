#!/bin/bash
OUT=gpurun_out/r02_tbmm_ncu; mkdir -p $OUT
timeout 300 python profiles/copy_floor.py > $OUT/copy_floor.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_nt" -s 1 -c 1 \
    -o $OUT/slab python profiles/ncu_ops.py tbmm > $OUT/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_nt" -s 1 -c 1 \
    -o $OUT/tiled python profiles/ncu_ops.py 'opts={"tile_sizes":[32,32,32],"thread_shape":[16,16,1],"block_shape":[1,1,1],"fusion_strategy":"max","rng_seed":0,"shared_memory_budget":49152,"unroll_copy_shared":false,"unroll_factor":1,"use_private":true,"use_shared":true}' tbmm > $OUT/ncu2.log 2>&1
cat $OUT/copy_floor.txt; tail -3 $OUT/ncu1.log $OUT/ncu2.log
