"""The bench step (TBMM || 2FCRelu || MLP3, forked onto side streams) with
alternative plans per operator: does a plan that is slower alone overlap
better? Device µs per step over graphs of NSTEP consecutive steps, plus each
variant alone. Usage: python profiles/step_variants.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1802_04730_b200 import ExecutionEngine  # noqa: E402

NSTEP = int(os.environ.get("NSTEP", "26"))

COMBOS = [  # r02: TBMM slab rows per warp in the step
    {"tbmm": {"tile_sizes": [4, 1, 2]}},
    {"tbmm": {"tile_sizes": [7, 1, 2]}},
    {"tbmm": {"tile_sizes": [9, 1, 2]}},
    {"tbmm": {"tile_sizes": [13, 1, 2]}},
    {"tbmm": {"tile_sizes": [5, 1, 2]}},
]

VARIANTS = {
    "2FCRelu": [None, {"tile_sizes": [4, 16, 1], "thread_shape": [64, 1, 1]}, {"tile_sizes": [2, 8, 1], "thread_shape": [32, 1, 1]},
                {"tile_sizes": [4, 4, 1], "thread_shape": [128, 1, 1]}, {"tile_sizes": [2, 16, 1], "thread_shape": [32, 1, 1]}],
    "MLP3": [None, {"tile_sizes": [2, 4, 1], "thread_shape": [32, 1, 1]}, {"tile_sizes": [4, 8, 1], "thread_shape": [64, 1, 1]},
             {"tile_sizes": [8, 4, 6], "thread_shape": [128, 1, 1]}, {"tile_sizes": [4, 2, 1], "thread_shape": [64, 1, 1]}],
}


def main():
    ee = ExecutionEngine()
    dev = torch.device("cuda", 0)
    ops = {n: bench.OpInstance(ee, torch, n, s, sd, NSTEP, dev, 1 + i) for i, (n, s, sd) in enumerate(bench.STEP_OPS)}
    main_s = torch.cuda.Stream()
    # PRIO="a,b,c": stream priorities of the tbmm / 2FCRelu / MLP3 side streams (lower = higher priority)
    prio = [int(x) for x in os.environ.get("PRIO", "0,0,0").split(",")]
    side = [torch.cuda.Stream(priority=p) for p in prio]

    def graph_of(group, pipelined=False):
        def body():
            if pipelined:  # consecutive steps overlap: each operator's stream runs its NSTEP steps, one join
                for sd in side[:len(group)]:
                    sd.wait_stream(main_s)
                for o, sd in zip(group, side):
                    with torch.cuda.stream(sd):
                        for k in range(NSTEP):
                            o.run(k)
                for sd in side[:len(group)]:
                    main_s.wait_stream(sd)
                return
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

    def timeit(g, n=40):
        with torch.cuda.stream(main_s):
            for _ in range(3):
                g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(main_s)
            for _ in range(n):
                g.replay()
            e1.record(main_s)
            e1.synchronize()
        return e0.elapsed_time(e1) * 1e3 / (n * NSTEP)

    base = {n: o.handle for n, o in ops.items()}
    for name, v in bench.STEP_PLANS.items():  # the bench's step plans
        o = ops[name]
        o.handle = base[name] = ee.compile(name, o.sets[0][0], o.sets[0][1],
                                           dict(ee.default_options(name, o.sets[0][0], o.sets[0][1]), **v))
    g0 = graph_of(list(ops.values()))
    print(f"default step {min(timeit(g0) for _ in range(8)):.2f} us", flush=True)
    import itertools
    for order in itertools.permutations(list(ops)) if os.environ.get("ORDER_ONLY") else []:
        g = graph_of([ops[n] for n in order])
        print(f"fork order {order}: {min(timeit(g) for _ in range(6)):.2f} us", flush=True)
    if os.environ.get("ORDER_ONLY"):
        return
    for name, v in [] if not os.environ.get("PIPE") else [("tbmm", {"tile_sizes": [7, 1, 2]}), ("tbmm", {"tile_sizes": [4, 1, 2]}),
                    ("2FCRelu", {"tile_sizes": [8, 8, 1], "thread_shape": [128, 1, 1]}),
                    ("2FCRelu", {"tile_sizes": [16, 8, 1], "thread_shape": [256, 1, 1]}),
                    ("MLP3", {"tile_sizes": [8, 4, 6], "thread_shape": [128, 1, 1]})]:
        o = ops[name]
        o.handle = ee.compile(name, o.sets[0][0], o.sets[0][1], dict(ee.default_options(name, o.sets[0][0], o.sets[0][1]), **v))
        gp = graph_of(list(ops.values()), pipelined=True)
        print(f"pipelined {name} {v}: {min(timeit(gp) for _ in range(5)):.2f} us per step", flush=True)
        o.handle = base[name]
    if os.environ.get("PIPE"):
        gp = graph_of(list(ops.values()), pipelined=True)
        print(f"pipelined steps {min(timeit(gp) for _ in range(8)):.2f} us per step", flush=True)
        for name in ops:
            print(f"{name} alone (back to back): {min(timeit(graph_of([ops[name]], pipelined=True)) for _ in range(3)):.2f} us", flush=True)
    if os.environ.get("PIPE_ONLY"):
        return
    combos = json.loads(os.environ["COMBOS_JSON"]) if os.environ.get("COMBOS_JSON") else COMBOS
    for combo in combos:
        try:
            for name, v in combo.items():
                o = ops[name]
                o.handle = ee.compile(name, o.sets[0][0], o.sets[0][1],
                                      dict(ee.default_options(name, o.sets[0][0], o.sets[0][1]), **v))
            gs = graph_of(list(ops.values()))
            step = min(timeit(gs) for _ in range(8))
            print(json.dumps({"combo": combo, "kernels": {n: ee.describe(o.handle)["kernel"] for n, o in ops.items()},
                              "step_us": round(step, 3)}), flush=True)
        except Exception as e:
            print(json.dumps({"combo": combo, "error": f"{type(e).__name__}: {e}"[:120]}), flush=True)
        for n, o in ops.items():
            o.handle = base[n]
    if os.environ.get("COMBOS_ONLY"):
        return
    for name, vs in VARIANTS.items():
        o = ops[name]
        for v in vs:
            try:
                o.handle = base[name] if v is None else ee.compile(
                    name, o.sets[0][0], o.sets[0][1], dict(ee.default_options(name, o.sets[0][0], o.sets[0][1]), **v))
                kern = ee.describe(o.handle)["kernel"]
                ga, gs = graph_of([o]), graph_of(list(ops.values()))
                alone = min(timeit(ga) for _ in range(3))
                step = min(timeit(gs) for _ in range(5))
                print(json.dumps({"op": name, "opts": v, "kernel": kern, "alone_us": round(alone, 3),
                                  "step_us": round(step, 3)}), flush=True)
            except Exception as e:  # a plan the op rejects
                print(json.dumps({"op": name, "opts": v, "error": f"{type(e).__name__}: {e}"[:120]}), flush=True)
        o.handle = base[name]


if __name__ == "__main__":
    main()
