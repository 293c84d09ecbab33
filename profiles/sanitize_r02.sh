#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over the kernels added or changed in round 2:
# FC cluster chains (column pairs, copies first), TMA-chunk FC, slab TBMM variants, tcgen05 GEMM
# (3xTF32 A in TMEM, fused two-layer FC), tcgen05 FC chain, TMA-halo gconv (small cases)
OUT=gpurun_out/r02_sanitizer; mkdir -p $OUT
export PYTHONFAULTHANDLER=1
# (16-CTA non-portable clusters excluded: synccheck reports "Missing wait" on ranks >= 8 and the
# instrumented kernel then faults; uninstrumented they are bit-exact in the GPU suite)
K_FFMA='(fc_chain_cluster or fc_tma or slab_variants or (golden and (mlp or fcrelu or tbmm))) and not 8-16-64'
K_TC='fc2_fused or fc_chains_tc or (gemm_tc and (shape0 or shape3 or shape5)) or tbmm_tc or (gconv_tc and shift and not paper)'
for tool in memcheck synccheck; do
  echo "== $tool ffma"; timeout 1500 compute-sanitizer --tool $tool --print-limit 6 python -m pytest tests/test_gpu_parity.py -q -k "$K_FFMA" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|Barrier error|at .*\.cu" | sort | uniq -c | head -12
  echo "== $tool tc"; timeout 1500 compute-sanitizer --tool $tool --print-limit 6 python -m pytest tests/test_gpu_tc.py -q -k "$K_TC" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|Barrier error|at .*\.cu" | sort | uniq -c | head -12
done > $OUT/memcheck_synccheck.txt 2>&1
cat $OUT/memcheck_synccheck.txt
echo "== racecheck ffma"; timeout 1500 compute-sanitizer --tool racecheck --print-limit 6 python -m pytest tests/test_gpu_parity.py -q -k "(fc_chain_cluster or slab_variants) and not 8-16-64" 2>&1 | grep -E "passed|failed|RACECHECK SUMMARY|hazard" | head -10 > $OUT/racecheck.txt
echo "== racecheck tc" >> $OUT/racecheck.txt; timeout 1500 compute-sanitizer --tool racecheck --print-limit 6 python -m pytest tests/test_gpu_tc.py -q -k "fc2_fused or fc_chains_tc or (gemm_tc and shape0)" 2>&1 | grep -E "passed|failed|RACECHECK SUMMARY|hazard" | head -10 >> $OUT/racecheck.txt
cat $OUT/racecheck.txt
echo "== synccheck + memcheck, the whole parity suite (16-CTA clusters excluded)" > $OUT/full.txt
for tool in synccheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 2 python -m pytest tests/test_gpu_parity.py -q -k "not 8-16-64 and not full_paper_shape and not pinned_host_large" 2>&1 | grep -E "passed|failed|ERROR SUMMARY" | sed "s/^/$tool: /" >> $OUT/full.txt
done
cat $OUT/full.txt
