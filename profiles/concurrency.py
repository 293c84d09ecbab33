"""Does the step's fork-join graph overlap its three operators? Times CUDA
graphs of: each op alone, the three serialised, the three forked onto
side streams (device time per replay, 200 replays, rotating inputs)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1802_04730_b200 import ExecutionEngine  # noqa: E402


def main():
    ee = ExecutionEngine()
    dev = torch.device("cuda", 0)
    ops = [bench.OpInstance(ee, torch, n, s, sd, 8, dev, 1 + i) for i, (n, s, sd) in enumerate(bench.STEP_OPS)]
    main_s = torch.cuda.Stream()
    side = [torch.cuda.Stream() for _ in range(3)]

    def capture(fn):
        gs = []
        with torch.cuda.stream(main_s):
            for i in range(8):
                fn(i)
            torch.cuda.synchronize()
            for i in range(8):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=main_s):
                    fn(i)
                gs.append(g)
        return gs

    def timeit(gs, n=200):
        with torch.cuda.stream(main_s):
            for i in range(10):
                gs[i % 8].replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(main_s)
            for i in range(n):
                gs[i % 8].replay()
            e1.record(main_s)
            e1.synchronize()
        return e0.elapsed_time(e1) * 1e3 / n

    for k, o in enumerate(ops):
        print(f"{o.name:8s} alone      {timeit(capture(lambda i, o=o: o.run(i))):8.2f} us/replay", flush=True)

    def serial(i):
        for o in ops:
            o.run(i)

    def forked(i):
        for sd in side:
            sd.wait_stream(main_s)
        for o, sd in zip(ops, side):
            with torch.cuda.stream(sd):
                o.run(i)
        for sd in side:
            main_s.wait_stream(sd)

    print(f"serial   3 ops      {timeit(capture(serial)):8.2f} us/replay")
    print(f"forked   3 ops      {timeit(capture(forked)):8.2f} us/replay")

    def tb2(i):  # tbmm twice, forked
        for sd in side[:2]:
            sd.wait_stream(main_s)
        for sd in side[:2]:
            with torch.cuda.stream(sd):
                ops[0].run(i)
        for sd in side[:2]:
            main_s.wait_stream(sd)
    print(f"forked   tbmm x2    {timeit(capture(tb2)):8.2f} us/replay")

    def pair(i, j):
        def f(k):
            for sd in side[:2]:
                sd.wait_stream(main_s)
            with torch.cuda.stream(side[0]):
                ops[i].run(k)
            with torch.cuda.stream(side[1]):
                ops[j].run(k)
            for sd in side[:2]:
                main_s.wait_stream(sd)
        return f
    for i, j in ((0, 1), (0, 2), (1, 2), (1, 0), (2, 0)):
        print(f"forked   {ops[i].name}+{ops[j].name:8s} {timeit(capture(pair(i, j))):8.2f} us/replay")

    # high-priority side streams for the FC chains (lower number = higher priority)
    lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
    pside = [torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=-1)]

    def forked_prio(k):
        for sd in pside:
            sd.wait_stream(main_s)
        for o, sd in zip(ops, pside):
            with torch.cuda.stream(sd):
                o.run(k)
        for sd in pside:
            main_s.wait_stream(sd)
    print(f"forked   3 ops, FC high priority {timeit(capture(forked_prio)):8.2f} us/replay")

    def forked_rev(k):
        for sd in side:
            sd.wait_stream(main_s)
        for o, sd in list(zip(ops, side))[::-1]:
            with torch.cuda.stream(sd):
                o.run(k)
        for sd in side:
            main_s.wait_stream(sd)
    print(f"forked   3 ops, reverse order   {timeit(capture(forked_rev)):8.2f} us/replay")


if __name__ == "__main__":
    main()
