"""Which of the step's operators overlap when forked onto side streams?
Each graph holds 8 consecutive steps (graph-launch cost amortised); times
are device µs per step. Also: two copies of one op, and MLP3 with a
non-cluster plan (rows=1, cn=1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1802_04730_b200 import ExecutionEngine  # noqa: E402

NSTEP = int(os.environ.get("NSTEP", "8"))


def main():
    ee = ExecutionEngine()
    dev = torch.device("cuda", 0)
    ops = {n: bench.OpInstance(ee, torch, n, s, sd, NSTEP, dev, 1 + i) for i, (n, s, sd) in enumerate(bench.STEP_OPS)}
    extra = bench.OpInstance(ee, torch, "MLP3", bench.STEP_OPS[2][1], bench.STEP_OPS[2][2], NSTEP, dev, 9)
    extra.handle = ee.compile("MLP3", extra.sets[0][0], extra.sets[0][1],
                              dict(ee.default_options("MLP3", extra.sets[0][0], extra.sets[0][1]),
                                   tile_sizes=[1, 1, 1], block_shape=[64, 1, 1]))
    ops["MLP3_nocluster"] = extra
    twin = {n: bench.OpInstance(ee, torch, n, s, sd, NSTEP, dev, 20 + i) for i, (n, s, sd) in enumerate(bench.STEP_OPS)}
    main_s = torch.cuda.Stream()
    side = [torch.cuda.Stream() for _ in range(3)]

    def graph_of(group):
        def body():
            for k in range(NSTEP):
                for sd in side[:len(group)]:
                    sd.wait_stream(main_s)
                for o, sd in zip(group, side):
                    with torch.cuda.stream(sd):
                        o.run(k)
                for sd in side[:len(group)]:
                    main_s.wait_stream(sd)
        with torch.cuda.stream(main_s):
            body()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=main_s):
                body()
        return g

    def timeit(g, n=100):
        with torch.cuda.stream(main_s):
            for _ in range(5):
                g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(main_s)
            for _ in range(n):
                g.replay()
            e1.record(main_s)
            e1.synchronize()
        return e0.elapsed_time(e1) * 1e3 / (n * NSTEP)

    cases = [["tbmm"], ["2FCRelu"], ["MLP3"], ["MLP3_nocluster"],
             ["tbmm", "2FCRelu"], ["tbmm", "MLP3"], ["2FCRelu", "MLP3"], ["tbmm", "MLP3_nocluster"],
             ["2FCRelu", "MLP3_nocluster"], ["tbmm", "2FCRelu", "MLP3"], ["tbmm", "2FCRelu", "MLP3_nocluster"]]
    for c in cases:
        print(f"{' || '.join(c):40s} {timeit(graph_of([ops[n] for n in c])):8.2f} us/step", flush=True)
    for n in ("tbmm", "2FCRelu", "MLP3"):
        print(f"{n + ' || ' + n:40s} {timeit(graph_of([ops[n], twin[n]])):8.2f} us/step", flush=True)
    def staged(first, then):  # fork `first` onto side streams, join, then `then` serially
        def body():
            for k in range(NSTEP):
                for sd in side[:len(first)]:
                    sd.wait_stream(main_s)
                for o, sd in zip(first, side):
                    with torch.cuda.stream(sd):
                        o.run(k)
                for sd in side[:len(first)]:
                    main_s.wait_stream(sd)
                for o in then:
                    o.run(k)
        with torch.cuda.stream(main_s):
            body()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=main_s):
                body()
        return g
    print(f"{'(tbmm || MLP3) -> 2FCRelu':40s} {timeit(staged([ops['tbmm'], ops['MLP3']], [ops['2FCRelu']])):8.2f} us/step",
          flush=True)
    print(f"{'2FCRelu -> (tbmm || MLP3)':40s} {timeit(staged([ops['2FCRelu']], [])) :8.2f} (2FCRelu alone, staged form)",
          flush=True)
    print(f"{'serial tbmm, MLP3, 2FCRelu':40s} {timeit(staged([], [ops['tbmm'], ops['MLP3'], ops['2FCRelu']])):8.2f} us/step",
          flush=True)
    for c in (["2FCRelu", "tbmm", "MLP3"], ["2FCRelu", "MLP3", "tbmm"], ["MLP3", "tbmm", "2FCRelu"],
              ["MLP3", "2FCRelu", "tbmm"]):
        print(f"{' || '.join(c) + ' (launch order)':40s} {timeit(graph_of([ops[n] for n in c])):8.2f} us/step",
              flush=True)


if __name__ == "__main__":
    main()
