#!/bin/bash
OUT=gpurun_out/r02p; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/read_floor profiles/read_floor.cu && /tmp/read_floor > $OUT/read_floor.txt 2>&1
python - >> $OUT/read_floor.txt 2>&1 <<'PY'
import torch
for n, dt in [(1 << 30, torch.bfloat16), (1 << 29, torch.float32), (53 << 20, torch.float32), (1 << 20, torch.float32)]:
    a = torch.empty(n, dtype=dt, device="cuda").uniform_(); b = torch.empty_like(a)
    for _ in range(3): b.copy_(a)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record(); b.copy_(a); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    by = 2 * n * a.element_size()
    print("torch copy %s %d MB: %.1f us %.1f GB/s (single pair, back to back)" % (dt, by >> 20, best * 1e3, by / best / 1e6))
    for nsets in (1, 2):
        src = [a] + [torch.empty_like(a).uniform_() for _ in range(nsets - 1)]
        dst = [b] + [torch.empty_like(b) for _ in range(nsets - 1)]
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for i in range(8):
                    dst[i % nsets].copy_(src[i % nsets])
            g.replay(); torch.cuda.synchronize()
            e0.record(s); g.replay(); e1.record(s); e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 8
        print("   graph of 8 copies over %d pair(s): %.1f us %.1f GB/s" % (nsets, us, by / us / 1e3))
        del src, dst, g
PY
cat $OUT/read_floor.txt
