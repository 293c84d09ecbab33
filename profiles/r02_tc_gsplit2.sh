#!/bin/bash
# r02: global vs cluster split-K at the same 128-wide tiles (TCB_TC_GSPLIT=1 forces the global path)
OUT=gpurun_out/r02_tc_gsplit2; mkdir -p $OUT
V='[{"tile_sizes":[128,128,32],"block_shape":[1,1,4]},{"tile_sizes":[128,112,32],"block_shape":[1,1,4]},{"tile_sizes":[128,128,32],"block_shape":[1,1,2]},{"tile_sizes":[128,64,32],"block_shape":[1,1,2]}]'
for m in tf32 3xtf32; do
  echo "== $m cluster"; timeout 300 python profiles/sweep.py tmm_huge "$V" $m 2>&1 | tail -5
  echo "== $m global"; TCB_TC_GSPLIT=1 timeout 300 python profiles/sweep.py tmm_huge "$V" $m 2>&1 | tail -5
done > $OUT/sweep.txt 2>&1; cat $OUT/sweep.txt
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -o $OUT/bn112 python profiles/ncu_ops.py reps=4 math=tf32 'opts={"tile_sizes":[128,112,32],"block_shape":[1,1,4]}' tmm_huge > $OUT/ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -o $OUT/bn128 python profiles/ncu_ops.py reps=4 math=tf32 'opts={"tile_sizes":[128,128,32],"block_shape":[1,1,4]}' tmm_huge >> $OUT/ncu.log 2>&1
tail -3 $OUT/ncu.log
