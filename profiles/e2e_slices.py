"""e2e step (bench.py's: TBMM + 2FCRelu + MLP3 through tcb_run with pinned
host buffers, 3 async calls on 3 streams, then all synchronised) at the
current TCB_HOST_SLICES; host wall clock per step, median of blocks."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1802_04730_b200 import ExecutionEngine  # noqa: E402


def main():
    ee = ExecutionEngine()
    dev = torch.device("cuda", 0)
    ops = [bench.OpInstance(ee, torch, n, s, sd, 1, dev, 1 + i, plan=bench.STEP_PLANS.get(n))
           for i, (n, s, sd) in enumerate(bench.STEP_OPS)]
    host = []
    for o in ops:
        ps, os_ = o.sets[0]
        hp = [x.cpu().pin_memory() for x in ps]
        ho = [x.cpu().pin_memory() for x in os_]
        plan = bench.STEP_PLANS.get(o.name)
        hh = ee.compile(o.name, hp, ho, dict(ee.default_options(o.name, hp, ho), **plan) if plan else None)
        host.append((o.name, hh, hp, ho))
    streams = [torch.cuda.Stream(device=dev) for _ in host]
    prepared = [ee.prepare(hh, hp, ho) for _, hh, hp, ho in host]

    def step(only=None):
        for k, (pr, st) in enumerate(zip(prepared, streams)):
            if only is None or k == only:
                pr.run(stream=st.cuda_stream, sync=False)
        for st in streams:
            st.synchronize()

    def timeit(only=None, n=200):
        for _ in range(300):
            step(only)
        blocks = []
        for _ in range(5):
            t0 = time.perf_counter()
            for _ in range(n):
                step(only)
            blocks.append((time.perf_counter() - t0) / n * 1e6)
        return sorted(blocks)[2]

    sl = os.environ.get("TCB_HOST_SLICES", "2")
    print(f"slices={sl}: step {timeit():.1f} us", " ".join(f"{h[0]} {timeit(k):.1f}" for k, h in enumerate(host)),
          flush=True)


if __name__ == "__main__":
    main()
