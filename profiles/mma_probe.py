import json, sys, torch
sys.path.insert(0, '/root/repo')
from paper_1802_04730_b200 import ExecutionEngine, options_baseline
ee = ExecutionEngine()
for M, N, K, bn in [(18944, 16, 144, 16), (18944, 16, 1152, 16), (18944, 128, 1152, 128), (18944, 32, 1152, 32)]:
    A = torch.rand(M, K, device='cuda'); B = torch.rand(N, K, device='cuda'); C = torch.zeros(M, N, device='cuda')
    o = json.loads(options_baseline(0)); o.update({"tile_sizes": [128, bn, 32], "block_shape": [1, 1, 1], "thread_shape": [256, 1, 1], "use_shared": True, "fusion_strategy": "min"})
    h = ee.compile("tmm", [A, B], [C], o, math="tf32")
    for _ in range(3): ee.run(h, [A, B], [C])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): ee.run(h, [A, B], [C])
    e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    kb = (K + 31) // 32
    print(f"M={M} N={N} K={K} bn={bn}: {us:.2f} us, {M//128} CTAs x {kb} k-blocks x 4 MMAs -> {us*1e3/(kb*4):.1f} ns per MMA per CTA")
