"""The paper's autotuner at paper shapes on one B200 (BASELINE configs[4]),
candidates costed on cold L2:
GA search over the kernel genes with measured device cost, the shape-keyed
cache it populates, and compile replaying the cached best (hit) with the
same bits. For each op: default plan time, tuned time, candidates, cache
hit on recompile. Usage: python profiles/tune_paper_r01.py [pop] [gens]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles"))

import torch  # noqa: E402

from ncu_ops import OPS  # noqa: E402
from paper_1802_04730_b200 import ExecutionEngine, options_baseline  # noqa: E402


def dev_time(ee, h, ps, os_, n=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            ee.run(h, ps, os_)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                ee.run(h, ps, os_, check_errors=False)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


def main():
    pop = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    gens = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    for key, math in (("c3", "ffma"), ("tbmm", "ffma"), ("gconv7", "ffma"), ("gconv14", "ffma"),
                      ("c3", "tf32"), ("mlp3", "ffma")):
        name, shapes, seeded = OPS[key]
        ee = ExecutionEngine()
        _, rets = ee.signature(name)
        oshapes = ee.infer_output_tensor_info(name, shapes, [seeded.get(i) for i in range(len(rets))])
        ps = [torch.rand(s, device="cuda") * 2 - 1 for s in shapes]
        os_ = [torch.rand(s, device="cuda") * 2 - 1 if i in seeded else torch.zeros(s, device="cuda")
               for i, s in enumerate(oshapes)]
        h0 = ee.compile(name, ps, os_, math=math)
        t_def = dev_time(ee, h0, ps, os_)
        k0 = ee.describe(h0)["kernel"]
        t_base, k_base = None, None
        if math == "ffma":  # the reference's baselineOptions(0) (options.cc:178-208) as compiled here
            try:
                hb = ee.compile(name, ps, os_, json.loads(options_baseline(0)))
                t_base, k_base = round(dev_time(ee, hb, ps, os_), 3), ee.describe(hb)["kernel"]
            except Exception as e:  # a baseline mapping this kernel family rejects
                k_base = f"{type(e).__name__}: {e}"[:80]
        t0 = time.perf_counter()
        r = ee.tune(name, ps, os_, population=pop, generations=gens, seed=1, math=math)
        wall = time.perf_counter() - t0
        hit = ee.cache_lookup(name, ps, os_) if math == "ffma" else None
        h1 = ee.compile(name, ps, os_, math=math)  # replays the cached best
        t_tuned = dev_time(ee, h1, ps, os_)
        out = {"op": key, "math": math, "baseline_options_us": t_base, "baseline_kernel": k_base,
               "default_us": round(t_def, 3), "default_kernel": k0,
               "tuned_us": round(t_tuned, 3), "tuned_kernel": ee.describe(h1)["kernel"],
               "speedup": round(t_def / t_tuned, 3), "tune_wall_s": round(wall, 1),
               "cache_hit_after": hit is not None if math == "ffma" else None}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
