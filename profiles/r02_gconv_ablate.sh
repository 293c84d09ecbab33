#!/bin/bash
# tcgen05 gconv ablations (TCB_GCONV_SKIP: 1 MMAs, 2 transposes, 4 output stores), paper shape TF32
for k in 0 7; do echo "skip=$k"; TCB_GCONV_SKIP=$k timeout 300 python profiles/sweep.py gconv '[]' tf32 2>&1 | head -1; done
timeout 300 python profiles/sweep.py gconv "[]" 3xtf32 2>\&1 | head -1
