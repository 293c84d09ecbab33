"""FC cluster kernel load modes vs the oracle on the paper 2FCRelu shape (debug)."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
from oracle_lib import Oracle
from paper_1802_04730_b200 import ExecutionEngine
orc = Oracle(); ee = ExecutionEngine(); rng = orc.rng(5)
I, W1, B1, W2, B2 = rng.f32((128, 1128)), rng.f32((128, 1128)), rng.f32((128,)), rng.f32((64, 128)), rng.f32((64,))
r1 = orc.fc_relu(I, W1, B1); r2 = orc.fc_relu(r1, W2, B2)
flush = torch.empty(64 << 20, device="cuda")
for ts in ([4, 8, 4], [4, 8, 1], [4, 8, 5], [4, 8, 3], [4, 8, 4], [4, 8, 1], [4, 8, 5], [4, 8, 3]):
    o = {"tile_sizes": ts, "thread_shape": [64, 1, 1], "fusion_strategy": "max", "use_shared": True}
    p = [torch.from_numpy(x).cuda() for x in (I, W1, B1, W2, B2)]
    out = [torch.zeros((128, 128), device="cuda"), torch.zeros((128, 64), device="cuda")]
    try:
        h = ee.compile("2FCRelu", p, out, dict(ee.default_options("2FCRelu", p, out), **o))
        flush.zero_(); torch.cuda.synchronize()
        ee.run(h, p, out); torch.cuda.synchronize()
        g1 = out[0].cpu().numpy()
        bad = np.argwhere(g1.view(np.uint32) != r1.view(np.uint32))
        print(ts, ee.describe(h)["kernel"], "O1 bad:", len(bad), bad[:6].tolist(), flush=True)
    except Exception as e:
        print(ts, "error", e, flush=True)
