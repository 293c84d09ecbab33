"""Runs selected paper operators a few times each at their paper shapes, for
ncu captures (profiles/README.md). Usage: python profiles/ncu_ops.py op [op ...]
ops: tmm tmm_big tmm_huge tbmm mlp1 2fcrelu mlp3 c3 kru gconv lut
(+ "opts=<json>", "math=ffma|tf32|3xtf32", "reps=N")"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1802_04730_b200 import ExecutionEngine  # noqa: E402

OPS = {
    "tmm": ("tmm", [(128, 32), (256, 32)], {}),
    "tmm_big": ("tmm", [(128, 1024), (1024, 1024)], {}),
    "tmm_huge": ("tmm", [(128, 16384), (4096, 16384)], {}),
    "tbmm": ("tbmm", [(500, 26, 72), (500, 26, 72)], {}),
    "mlp1": ("MLP1", [(128, 1128), (128, 1128), (128,)], {}),
    "2fcrelu": ("2FCRelu", [(128, 1128), (128, 1128), (128,), (64, 128), (64,)], {}),
    "mlp3": ("MLP3", [(128, 128), (64, 128), (64,), (32, 64), (32,), (2, 32), (2,)], {0: (128, 128)}),
    "c3": ("C3", [(128, 1024), (1000, 1024)], {0: (128, 1000)}),
    "kru": ("3KRU", [(32, 16), (32, 16), (32, 16), (256, 16, 16, 16)], {}),
    "gconv": ("gconv", [(32, 32, 16, 58, 58), (32, 16, 16, 3, 3), (16,)], {}),
    "gconv14": ("gconv", [(32, 32, 16, 16, 16), (32, 16, 16, 3, 3), (16,)], {}),
    "gconv7": ("gconv", [(32, 32, 32, 9, 9), (32, 32, 32, 3, 3), (32,)], {}),
    "gconv56": ("gconv", [(32, 32, 4, 58, 58), (32, 4, 4, 3, 3), (4,)], {}),
    "gconv28": ("gconv", [(32, 32, 8, 30, 30), (32, 8, 8, 3, 3), (8,)], {}),
    "lut": ("2LUT", [(10_000_000, 64), (128, 50), (10_000_000, 64), (128, 50)], {}),
}


def main():
    ee = ExecutionEngine()
    opts = None
    reps = 3
    math = "ffma"
    for a in sys.argv[1:]:
        if a.startswith("opts="):
            opts = json.loads(a[5:])
            continue
        if a.startswith("math="):
            math = a[5:]
            continue
        if a.startswith("reps="):
            reps = int(a[5:])
            continue
        name, shapes, seeded = OPS[a]
        ps = []
        for i, s in enumerate(shapes):
            if name == "2LUT" and i in (1, 3):
                ps.append(torch.randint(0, shapes[i - 1][0], s, device="cuda", dtype=torch.int32))
            else:
                ps.append(torch.rand(s, device="cuda") * 2 - 1)
        _, rets = ee.signature(name)
        given = [seeded.get(i) for i in range(len(rets))]
        oshapes = ee.infer_output_tensor_info(name, shapes, given)
        outs = [torch.rand(s, device="cuda") for s in oshapes]
        o = dict(ee.default_options(name, ps, outs), **opts) if opts else None  # as bench.py's STEP_PLANS
        h = ee.compile(name, ps, outs, o, math=math)
        print(a, ee.describe(h)["kernel"], flush=True)
        for _ in range(reps):
            ee.run(h, ps, outs)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
