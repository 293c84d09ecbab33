"""Practical HBM floor for a kernel of a given traffic: device time of a
torch copy (read n/2 bytes + write n/2 bytes) rotating over buffers larger
than 2x L2, back to back in a CUDA graph. Usage: python profiles/copy_floor.py"""
import torch

L2 = 126 << 20
s = torch.cuda.Stream()
print("traffic_MB  us_per_copy  GB/s")
for mb in [0.16, 1.22, 5.64, 8.84, 20.0, 88.1, 426.3]:
    half = int(mb * 1e6 / 2) // 16 * 4
    nsets = max(2, min(64, int(2 * L2 / (mb * 1e6)) + 1))
    src = [torch.empty(half, device="cuda").uniform_() for _ in range(nsets)]
    dst = [torch.empty(half, device="cuda") for _ in range(nsets)]
    with torch.cuda.stream(s):
        for a, b in zip(src, dst):
            b.copy_(a)
        torch.cuda.synchronize()
        per = max(nsets, 32)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(per):
                dst[i % nsets].copy_(src[i % nsets])
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5):
            g.replay()
        e1.record(s)
        e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (5 * per)
    print(f"{mb:9.2f}  {us:10.3f}  {2 * half * 4 / us / 1e3:8.1f}", flush=True)
    del src, dst
