"""The production model (prodmodel.py) at the paper's sizes: per-kernel device
times of one forward (ncu launch list of 5 eager forwards), and the graph's
time per forward, to see where the chain's 69 us go."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1802_04730_b200 import ExecutionEngine  # noqa: E402
from paper_1802_04730_b200.prodmodel import PAPER_SIZES  # noqa: E402
from paper_1802_04730_b200.prodmodel import ProductionModel  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    ee = ExecutionEngine()
    S = dict(PAPER_SIZES)
    if os.environ.get("PM_E"):  # smaller tables: is the bimodal forward time a table-size (TLB) effect?
        S["E1"] = S["E2"] = int(os.environ["PM_E"])
    g = torch.Generator(device=dev)
    g.manual_seed(21)
    r = lambda *sh: torch.rand(sh, generator=g, device=dev) * 2 - 1  # noqa: E731
    p = dict(LUT1=r(S["E1"], S["D"]), LUT2=r(S["E2"], S["D"]),
             I1=torch.randint(0, S["E1"], (S["B"], S["L1"]), generator=g, device=dev, dtype=torch.int32),
             I2=torch.randint(0, S["E2"], (S["B"], S["L2"]), generator=g, device=dev, dtype=torch.int32),
             I3=r(S["B"], S["WX"]), W=r(S["WY"], S["WX"]), W1=r(S["N"], 2 * S["D"] + S["WY"]), B1=r(S["N"]),
             W2=r(S["O"], S["N"]), B2=r(S["O"]), W3=r(S["P"], S["O"]), B3=r(S["P"]), W4=r(S["Q"], S["P"]),
             B4=r(S["Q"]))
    m = ProductionModel(ee, p, fork=bool(os.environ.get("PM_FORK")))
    print({k: v for k, v in m.kernels.items()}, flush=True)
    if os.environ.get("EAGER"):
        for _ in range(5):
            m.forward_eager()
        torch.cuda.synchronize()
        return
    with torch.cuda.stream(m.stream):
        for b in range(0 if os.environ.get('PM_E') else 6):  # the same launches without the graph
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(m.stream)
            for _ in range(100):
                m._enqueue(check_errors=False)
            e1.record(m.stream)
            e1.synchronize()
            print(f"eager block {b}: {e0.elapsed_time(e1) * 10:.1f} us per forward (device)", flush=True)
    m.capture()
    for _ in range(5):
        m.replay()
    torch.cuda.synchronize()
    import bench  # noqa: E402  (its NVML clock sampler)
    for b in range(10):  # consecutive blocks: does the rate drift as replays go on? (+ SM clocks)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with bench.ClockSampler(dev) as cs:
            e0.record(m.stream)
            t0 = time.perf_counter()
            for _ in range(1000):
                m.replay()
            t1 = time.perf_counter()
            e1.record(m.stream)
            while not e1.query():
                time.sleep(0.0005)
        c = cs.summary()
        print(f"graph block {b}: {e0.elapsed_time(e1):.1f} us per forward (device), "
              f"host enqueue {(t1 - t0) * 1e3:.1f} us per replay, sm {c['sm_mhz']} MHz "
              f"(min {min(cs.samples) if cs.samples else None}, {c['samples']} samples) {c['reasons']}", flush=True)


if __name__ == "__main__":
    main()
