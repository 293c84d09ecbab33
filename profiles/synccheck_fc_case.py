import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1802_04730_b200 import ExecutionEngine
rows, cn, thr, B, K, N1, N2 = [int(x) for x in sys.argv[1:8]]
ee = ExecutionEngine()
rng = np.random.default_rng(0)
f = lambda *s: torch.from_numpy(rng.uniform(-1, 1, s).astype(np.float32)).cuda()
ins = [f(B, K), f(N1, K), f(N1), f(N2, N1), f(N2)]
outs = [torch.zeros(B, N1, device='cuda'), torch.zeros(B, N2, device='cuda')]
o = {"block_shape": [1, 1, 1], "fusion_strategy": "max", "rng_seed": 0, "shared_memory_budget": 49152,
     "thread_shape": [thr, 1, 1], "tile_sizes": [rows, cn, 1], "unroll_copy_shared": False, "unroll_factor": 1,
     "use_private": False, "use_shared": True}
h = ee.compile("2FCRelu", ins, outs, o)
ee.run(h, ins, outs); torch.cuda.synchronize()
print(sys.argv[1:], ee.describe(h)["kernel"], "ok")
