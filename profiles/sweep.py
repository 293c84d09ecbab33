"""Time one paper operator under several MappingOptions (device time per
launch, CUDA graph of back-to-back launches, L2-rotated inputs).
Usage: python profiles/sweep.py tbmm '[{"tile_sizes":[2,2,1]}, ...]' [math]
Each dict is merged over the op's default options."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles"))

import torch  # noqa: E402

from ncu_ops import OPS  # noqa: E402
from paper_1802_04730_b200 import ExecutionEngine  # noqa: E402


def main():
    key, variants = sys.argv[1], json.loads(sys.argv[2])
    math = sys.argv[3] if len(sys.argv) > 3 else "ffma"
    name, shapes, seeded = OPS[key]
    ee = ExecutionEngine()
    _, rets = ee.signature(name)
    oshapes = ee.infer_output_tensor_info(name, shapes, [seeded.get(i) for i in range(len(rets))])
    nsets = 16
    sets = []
    for _ in range(nsets):
        ps = [torch.randint(0, shapes[i - 1][0], s, device="cuda", dtype=torch.int32)
              if name == "2LUT" and i in (1, 3) else torch.rand(s, device="cuda") * 2 - 1
              for i, s in enumerate(shapes)]
        sets.append((ps, [torch.rand(s, device="cuda") for s in oshapes]))
    base = ee.default_options(name, sets[0][0], sets[0][1])
    s = torch.cuda.Stream()
    for v in [{}] + variants:
        o = dict(base)
        o.update(v)
        if not v and math != "ffma":
            o = None  # the tensor-core plan (no explicit options)
        try:
            h = ee.compile(name, sets[0][0], sets[0][1], o, math=math)
            desc = ee.describe(h)["kernel"]
            with torch.cuda.stream(s):
                for p, q in sets:
                    ee.run(h, p, q)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for r in range(4):
                        for p, q in sets:
                            ee.run(h, p, q, check_errors=False)
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(5):
                    g.replay()
                e1.record(s)
                e1.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (5 * 4 * nsets)
            print(f"{us:9.3f} us  {desc:50s} {json.dumps(v)}", flush=True)
        except Exception as e:
            print(f"   error   {json.dumps(v)}: {e}", flush=True)


if __name__ == "__main__":
    main()
