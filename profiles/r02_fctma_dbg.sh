OUT=gpurun_out/fctma_dbg; mkdir -p $OUT
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "test_fc_tma_variants and 8-8-128" > $OUT/memcheck.log 2>&1
tail -60 $OUT/memcheck.log
