# tcgen05 GEMM with whole-warp elect.sync MMA issue: tolerance tests + timings
timeout 400 python -m pytest tests/test_gpu_tc.py -x -q -k "not gconv and not kru" 2>&1 | tail -1
for op in tmm_huge c3 tbmm tmm; do for m in tf32 3xtf32; do echo "$op $m $(timeout 100 python profiles/sweep.py $op '[]' $m 2>&1 | tail -1 | cut -c1-60)"; done; done
