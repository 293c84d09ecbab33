B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTCB_DEBUG_BARRIERS -I paper_1802_04730_b200/csrc profiles/tc_gconv_debug.cu"
$B -DTCB_DBG_NO_MMA -DTCB_DBG_NO_TMA -DTCB_DBG_NO_LDTM -o /tmp/t1 && echo "== no mma/tma/ldtm" && /tmp/t1 0 2>&1 | head -3
$B -DTCB_DBG_NO_MMA -DTCB_DBG_NO_TMA -o /tmp/t2 && echo "== no mma/tma" && /tmp/t2 0 2>&1 | head -3
$B -DTCB_DBG_NO_MMA -DTCB_DBG_NO_LDTM -o /tmp/t3 && echo "== no mma/ldtm" && /tmp/t3 0 2>&1 | head -3
$B -DTCB_DBG_NO_LDTM -o /tmp/t4 && echo "== no ldtm" && /tmp/t4 0 2>&1 | head -3
$B -o /tmp/t5 && echo "== all" && /tmp/t5 0 2>&1 | head -3
