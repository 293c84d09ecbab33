"""Stress the fused FC-chain kernel: many launches per configuration,
reporting the first failure (the kernel traps instead of hanging when an
mbarrier phase never completes). Usage: python profiles/fc_stress.py [n]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1802_04730_b200 import ExecutionEngine  # noqa: E402

CFG = {
    "MLP3": ([(128, 128), (64, 128), (64,), (32, 64), (32,), (2, 32), (2,)], {0: (128, 128)}),
    "2FCRelu": ([(128, 1128), (128, 1128), (128,), (64, 128), (64,)], {}),
    "MLP1": ([(128, 1128), (128, 1128), (128,)], {}),
}


def opts(rows, cn, threads):
    return {"block_shape": [1, 1, 1], "fusion_strategy": "max", "rng_seed": 0, "shared_memory_budget": 49152,
            "thread_shape": [threads, 1, 1], "tile_sizes": [rows, cn, 1], "unroll_copy_shared": False,
            "unroll_factor": 1, "use_private": False, "use_shared": True}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    ee = ExecutionEngine()
    s = torch.cuda.Stream()
    runs = [(k, None) for k in CFG] + [("MLP3", opts(r, c, t)) for r, c, t in
                                       [(1, 1, 64), (4, 1, 64), (1, 4, 64), (4, 2, 64), (2, 4, 64), (4, 4, 128)]]
    for name, o in runs:
        shapes, seeded = CFG[name]
        ps = [torch.rand(sh, device="cuda") for sh in shapes]
        _, rets = ee.signature(name)
        osh = ee.infer_output_tensor_info(name, shapes, [seeded.get(i) for i in range(len(rets))])
        outs = [torch.rand(sh, device="cuda") for sh in osh]
        h = ee.compile(name, ps, outs, o)
        t0 = time.time()
        try:
            with torch.cuda.stream(s):
                for i in range(n):
                    ee.run(h, ps, outs)
                    if i % 50 == 0:
                        torch.cuda.synchronize()
            torch.cuda.synchronize()
        except Exception as e:
            print(f"{name} {o and o['tile_sizes']} {o and o['thread_shape']}: FAILED {e}", flush=True)
            return
        print(f"{name}: {n} launches ok in {time.time() - t0:.2f}s ({ee.describe(h)['kernel']})", flush=True)


if __name__ == "__main__":
    main()
