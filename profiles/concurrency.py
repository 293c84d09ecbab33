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


if __name__ == "__main__":
    main()
