# tcgen05 3-KRU: tolerance tests (both d2 chunks), then paper-shape timings vs the FFMA kernel
mkdir -p gpurun_out
for dc in 8 16; do
  TCB_KRU_DC=$dc timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "kru" 2>&1 | tail -1
  for m in tf32 3xtf32; do echo "dc=$dc $m $(TCB_KRU_DC=$dc timeout 100 python profiles/sweep.py kru '[]' $m 2>&1 | tail -1 | cut -c1-12)"; done
done
