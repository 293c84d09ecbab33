"""The production model (prodmodel.py) at the paper's sizes: per-kernel device
times of one forward (ncu launch list of 5 eager forwards), and the graph's
time per forward, to see where the chain's 69 us go."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1802_04730_b200 import ExecutionEngine  # noqa: E402
from paper_1802_04730_b200.prodmodel import PAPER_SIZES as S  # noqa: E402
from paper_1802_04730_b200.prodmodel import ProductionModel  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    ee = ExecutionEngine()
    g = torch.Generator(device=dev)
    g.manual_seed(21)
    r = lambda *sh: torch.rand(sh, generator=g, device=dev) * 2 - 1  # noqa: E731
    p = dict(LUT1=r(S["E1"], S["D"]), LUT2=r(S["E2"], S["D"]),
             I1=torch.randint(0, S["E1"], (S["B"], S["L1"]), generator=g, device=dev, dtype=torch.int32),
             I2=torch.randint(0, S["E2"], (S["B"], S["L2"]), generator=g, device=dev, dtype=torch.int32),
             I3=r(S["B"], S["WX"]), W=r(S["WY"], S["WX"]), W1=r(S["N"], 2 * S["D"] + S["WY"]), B1=r(S["N"]),
             W2=r(S["O"], S["N"]), B2=r(S["O"]), W3=r(S["P"], S["O"]), B3=r(S["P"]), W4=r(S["Q"], S["P"]),
             B4=r(S["Q"]))
    m = ProductionModel(ee, p)
    print({k: v for k, v in m.kernels.items()}, flush=True)
    if os.environ.get("EAGER"):
        for _ in range(5):
            m.forward_eager()
        torch.cuda.synchronize()
        return
    m.capture()
    for _ in range(5):
        m.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.stream)
    for _ in range(100):
        m.replay()
    e1.record(m.stream)
    e1.synchronize()
    print(f"graph: {e0.elapsed_time(e1) * 10:.1f} us per forward", flush=True)


if __name__ == "__main__":
    main()
