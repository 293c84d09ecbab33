"""Production model graph: one stream vs C3 forked beside 2LUT (device us per
forward, 8 blocks of 200 replays each, to see whether the fork is bimodal)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1802_04730_b200 import ExecutionEngine  # noqa: E402
from paper_1802_04730_b200.prodmodel import PAPER_SIZES as S  # noqa: E402
from paper_1802_04730_b200.prodmodel import ProductionModel  # noqa: E402


def main():
    ee = ExecutionEngine()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(21)
    r = lambda *sh: torch.rand(sh, generator=g, device=dev) * 2 - 1  # noqa: E731
    p = dict(LUT1=r(S["E1"], S["D"]), LUT2=r(S["E2"], S["D"]),
             I1=torch.randint(0, S["E1"], (S["B"], S["L1"]), generator=g, device=dev, dtype=torch.int32),
             I2=torch.randint(0, S["E2"], (S["B"], S["L2"]), generator=g, device=dev, dtype=torch.int32),
             I3=r(S["B"], S["WX"]), W=r(S["WY"], S["WX"]), W1=r(S["N"], 2 * S["D"] + S["WY"]), B1=r(S["N"]),
             W2=r(S["O"], S["N"]), B2=r(S["O"]), W3=r(S["P"], S["O"]), B3=r(S["P"]), W4=r(S["Q"], S["P"]),
             B4=r(S["Q"]))
    for fork in (False, True):
        m = ProductionModel(ee, p, fork=fork).capture()
        for _ in range(100):
            m.replay()
        blocks = []
        for _ in range(8):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(m.stream)
            for _ in range(200):
                m.replay()
            e1.record(m.stream)
            e1.synchronize()
            blocks.append(round(e0.elapsed_time(e1) * 1e3 / 200, 2))
        print(f"fork={fork}: us per forward by block {blocks}", flush=True)


if __name__ == "__main__":
    main()
