#!/usr/bin/env python
"""tc-b200 benchmark — BASELINE.json configs[1] on B200.

A step is one pass of the hot path over one batch of synthetic input:
    TBMM     Z(b,n,k) +=! X(b,n,m) * Y(b,k,m)       B=500, N=26, M=72, K=26
    2FCRelu  O1 = relu(I W1^T + B1), O2 = relu(O1 W2^T + B2)   B=128, 1128 -> 128 -> 64
    MLP3     O2..O4 = three FC+ReLU layers from O1    B=128, 128 -> 64 -> 32 -> 2
each a call of the TC definition through the C ABI (libtcb.so). `value` is
whole-job GFLOP/s (algorithmic FLOPs of all ranks / max-over-ranks device
time); `e2e` is the same metric through tcb_run with pinned HOST buffers
(H2D + kernels + D2H inside the timed region). Weak scaling: every rank runs
its own batch (batch sharding of a global batch of N x 500 / N x 128), no
collective on the data path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "µs/call and GFLOP/s per TC op at paper shapes (1/2/4/8 B200) vs roofline & CPU ref"
L2_BYTES = 126 * 1024 * 1024

# (def, parameter shapes, seeded return shapes) — BASELINE.md §2
STEP_OPS = [
    ("tbmm", [(500, 26, 72), (500, 26, 72)], {}),
    ("2FCRelu", [(128, 1128), (128, 1128), (128,), (64, 128), (64,)], {}),
    ("MLP3", [(128, 128), (64, 128), (64,), (32, 64), (32,), (2, 32), (2,)], {0: (128, 128)}),
]
# every paper operator at its paper shape (per-op table)
PAPER_OPS = [
    ("tmm", "tmm 128x256x32", [(128, 32), (256, 32)], {}),
    ("tmm", "tmm 128x1024x1024", [(128, 1024), (1024, 1024)], {}),
    ("tbmm", "tbmm 500,26,72,26", [(500, 26, 72), (500, 26, 72)], {}),
    ("MLP1", "MLP1 128x1128->128", [(128, 1128), (128, 1128), (128,)], {}),
    ("2FCRelu", "2FCRelu 128x1128->128->64", [(128, 1128), (128, 1128), (128,), (64, 128), (64,)], {}),
    ("MLP3", "MLP3 128->64->32->2", [(128, 128), (64, 128), (64,), (32, 64), (32,), (2, 32), (2,)],
     {0: (128, 128)}),
    ("C3", "C3 128x1024->1000", [(128, 1024), (1000, 1024)], {0: (128, 1000)}),
    ("3KRU", "3KRU M=256 16^3->32^3", [(32, 16), (32, 16), (32, 16), (256, 16, 16, 16)], {}),
    ("gconv", "gconv 32,32,16,16,58x58,3x3", [(32, 32, 16, 58, 58), (32, 16, 16, 3, 3), (16,)], {}),
    ("2LUT", "2LUT E=1e7,D=64,B=128,L=50",
     [(10_000_000, 64), (128, 50), (10_000_000, 64), (128, 50)], {}),
]
INT_PARAMS = {"2LUT": {1, 3}, "1LUT": {1}}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# --------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None
        self.lines = []

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None
        return self

    def _read(self):
        for line in self.p.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- workload
class OpInstance:
    """One TC op bound to device tensors (a rotating set of input copies)."""

    def __init__(self, ee, torch, name, pshapes, seeded, nsets, dev, seed, host_init=True):
        self.ee, self.torch, self.name = ee, torch, name
        _, rets = ee.signature(name)
        ints = INT_PARAMS.get(name, set())
        given = [seeded.get(i) for i in range(len(rets))]
        oshapes = ee.infer_output_tensor_info(name, [tuple(s) for s in pshapes], given)
        self.pshapes, self.oshapes = pshapes, oshapes
        self.inout = set(seeded)
        self.sets = []
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        for k in range(nsets):
            ps = []
            for i, s in enumerate(pshapes):
                if i in ints:  # LUT row indices in [0, E) of the table they index
                    ps.append(torch.randint(0, pshapes[i - 1][0], s, generator=g, device=dev,
                                            dtype=torch.int32))
                else:
                    ps.append(torch.rand(s, generator=g, device=dev) * 2 - 1)
            os_ = [torch.rand(s, generator=g, device=dev) * 2 - 1 if i in self.inout else
                   torch.zeros(s, device=dev) for i, s in enumerate(oshapes)]
            self.sets.append((ps, os_))
        self.handle = ee.compile(name, self.sets[0][0], self.sets[0][1])
        d = ee.describe(self.handle)
        self.flops, self.bytes, self.kernel = d["flops"], d["bytes"], d["kernel"]

    def run(self, k, check=False):
        ps, os_ = self.sets[k % len(self.sets)]
        self.ee.run(self.handle, ps, os_, check_errors=check)

    def set_bytes(self):
        t = 0
        for ps, os_ in self.sets[:1]:
            t += sum(x.numel() * 4 for x in ps) + sum(x.numel() * 4 for x in os_)
        return t


def time_device(torch, fn, iters, stream):
    """Device time of `iters` calls of fn(i) on `stream`, via CUDA events."""
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record(stream)
    for i in range(iters):
        fn(i)
    e.record(stream)
    e.synchronize()
    return s.elapsed_time(e) * 1e-3  # seconds


# ----------------------------------------------------------- CPU baseline
def cpu_reference_sample(threads=None, scale=16):
    """The reference's own CPU implementation of the path — the interpreter
    backend::interpretReference of the reference library (oracle/_ref, built
    from /root/reference) — on a bounded sample of the step: 1/scale of
    every batch, rows split across host threads (reentrant per
    interpreter.h:78). Falls back to the C restatement (OpenMP) when the
    reference build is absent. Returns (GFLOP/s, seconds, info dict)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import concurrent.futures as cf

    from oracle_lib import Oracle, RefLib

    orc = Oracle()
    src = open(os.path.join(ROOT, "paper_1802_04730_b200", "tc", "ops.tc")).read()
    rng = orc.rng(7)
    tb = 500 // scale  # TBMM batches
    fb = max(1, 128 // scale)  # FC rows
    X, Y = rng.f32((tb, 26, 72)), rng.f32((tb, 26, 72))
    I, W1, B1 = rng.f32((fb, 1128)), rng.f32((128, 1128)), rng.f32((128,))
    W2, B2 = rng.f32((64, 128)), rng.f32((64,))
    O1 = rng.f32((fb, 128))
    M2, C2, M3, C3b, M4, C4 = (rng.f32((64, 128)), rng.f32((64,)), rng.f32((32, 64)), rng.f32((32,)),
                               rng.f32((2, 32)), rng.f32((2,)))
    flops = 2.0 * tb * 26 * 26 * 72 + 2.0 * fb * (128 * 1128 + 64 * 128) + 2.0 * fb * (
        64 * 128 + 32 * 64 + 2 * 32)
    threads = threads or os.cpu_count() or 1
    if RefLib.available():
        ref = RefLib()
        jobs = []
        for b in range(tb):
            jobs.append(("tbmm", {"X": X[b:b + 1], "Y": Y[b:b + 1]}, ["Z"]))
        for r in range(fb):
            jobs.append(("2FCRelu", {"I": I[r:r + 1], "W1": W1, "B1": B1, "W2": W2, "B2": B2}, ["O1", "O2"]))
            jobs.append(("MLP3", {"I": O1[r:r + 1], "W2": M2, "B2": C2, "W3": M3, "B3": C3b, "W4": M4,
                                  "B4": C4, "O1": O1[r:r + 1]}, ["O2", "O3", "O4"]))
        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda j: ref.run(src, j[0], j[1], j[2]), jobs))
        dt = time.perf_counter() - t0
        kind = "reference"
    else:
        orc.lib.orc_set_threads(threads)
        t0 = time.perf_counter()
        orc.tbmm(X, Y)
        o1 = orc.fc_relu(I, W1, B1)
        orc.fc_relu(o1, W2, B2)
        orc.mlp3(O1, M2, C2, M3, C3b, M4, C4)
        dt = time.perf_counter() - t0
        kind = "port"
    info = {"kind": kind, "cores": threads,
            "sample": f"1/{scale} of the step's batches: TBMM B={tb}, 2FCRelu B={fb}, MLP3 B={fb} "
                      f"({flops / 1e6:.2f} MFLOP)"}
    return flops / dt / 1e9, dt, info


def reference_arm(args, rank, world):
    if rank != 0:
        return
    scale = 16
    for _ in range(args.warmup):
        cpu_reference_sample(scale=scale)
    vals, times = [], []
    info = None
    for _ in range(args.steps):
        v, dt, info = cpu_reference_sample(scale=scale)
        vals.append(v)
        times.append(dt)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(statistics.median(times) * 1e3 * scale, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "TBMM(B=500,N=26,M=72,K=26) + 2FCRelu(B=128,1128->128->64) + "
                               "MLP3(B=128,128->64->32->2) per step", "parallelism": f"dp{args.gpus}",
                   "note": "reference CPU interpreter on a bounded 1/16 sample per step; ms_per_step "
                           "extrapolated to the full step"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", **info},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- main arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="tcb", choices=["tcb", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ops", action="store_true", help="skip the per-op paper table")
    ap.add_argument("--profile-only", action="store_true", help="run a few steps, print nothing (ncu)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_1802_04730_b200 import ExecutionEngine, device_info

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    peaks, peak_src = load_peaks()
    ee = ExecutionEngine()

    # rotating input sets larger than L2 (inputs AND weights rotate)
    probe = [OpInstance(ee, torch, n, s, sd, 1, dev, 0) for n, s, sd in STEP_OPS]
    set_bytes = sum(o.set_bytes() for o in probe)
    nsets = max(2, int(np.ceil(2 * L2_BYTES / set_bytes)))
    ops = [OpInstance(ee, torch, n, s, sd, nsets, dev, 1 + i + 100 * rank) for i, (n, s, sd) in
           enumerate(STEP_OPS)]
    del probe
    flops_step = sum(o.flops for o in ops)
    stream = torch.cuda.Stream(device=dev)

    with torch.cuda.stream(stream):
        def step(i):
            for o in ops:
                o.run(i)

        # capture one CUDA graph per input set (3 launches each)
        for i in range(nsets):
            step(i)
        torch.cuda.synchronize()
        graphs = []
        for i in range(nsets):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(i)
            graphs.append(g)
        for i in range(args.warmup):
            graphs[i % nsets].replay()
        torch.cuda.synchronize()
        if args.profile_only:
            for i in range(args.steps):
                graphs[i % nsets].replay()
            torch.cuda.synchronize()
            return

        # ---- timed region: K steps, barrier + sync both sides, max over ranks
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            el = time_device(torch, lambda i: graphs[i % nsets].replay(), args.steps, stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            t = torch.tensor([el], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        value = world * flops_step * args.steps / el / 1e9
        ms_step = el / args.steps * 1e3

        # ---- per-op device time inside the step (same stream, L2-rotated):
        # one graph launches the op on every rotating input set back to back
        per_op = []
        for o in ops:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for i in range(nsets):
                    o.run(i)
            for i in range(3):
                g.replay()
            reps = max(4, args.steps // nsets)
            t = time_device(torch, lambda i: g.replay(), reps, stream) / (reps * nsets)
            per_op.append((o, t))

        # ---- e2e: tcb_run with pinned HOST buffers (H2D + kernel + D2H per call)
        host = []
        h2d = d2h = 0
        for o in ops:
            ps, os_ = o.sets[0]
            hp = [x.cpu().pin_memory() for x in ps]
            ho = [x.cpu().pin_memory() for x in os_]
            hh = ee.compile(o.name, hp, ho)
            host.append((hh, hp, ho))
            h2d += sum(x.numel() * 4 for x in hp) + sum(x.numel() * 4 for i, x in enumerate(ho) if i in o.inout)
            d2h += sum(x.numel() * 4 for x in ho)

        def e2e_step(i):
            for hh, hp, ho in host:
                ee.run(hh, hp, ho, stream=stream.cuda_stream)

        for i in range(args.warmup):
            e2e_step(i)
        ke = max(20, args.steps // 4)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_dev = time_device(torch, e2e_step, ke, stream)
        e2e_wall = time.perf_counter() - t0
        e2e_t = max(e2e_dev, e2e_wall)
        if world > 1:
            t = torch.tensor([e2e_t], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_t = float(t.item())
        e2e_value = world * flops_step * ke / e2e_t / 1e9

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant (largest-share) kernel of the step
    step_dev = sum(t for _, t in per_op)
    dom, dom_t = max(per_op, key=lambda x: x[1])
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = dom.bytes / dom_t / 1e9
    roofline = {"bound": "hbm", "kernel": f"{dom.name}: {dom.kernel}", "achieved": round(achieved, 1),
                "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": None,
                "algorithmic_bytes": int(dom.bytes), "launch_us": round(dom_t * 1e6, 3),
                "share_of_step": round(dom_t / step_dev, 3), "peak_source": peak_src,
                "note": "FFMA-exact fp32 kernels: no tensor-core roofline applies; HBM roofline over the "
                        "kernel's algorithmic bytes (inputs once, outputs once)"}
    tbmm = [x for x in per_op if x[0].name == "tbmm"][0]
    roofline_ops = {
        o.name: {"us": round(t * 1e6, 3), "gflops": round(o.flops / t / 1e9, 1),
                 "hbm_gbs": round(o.bytes / t / 1e9, 1), "hbm_frac": round(o.bytes / t / 1e9 / hbm_peak, 4),
                 "share": round(t / step_dev, 3), "kernel": o.kernel} for o, t in per_op}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (U[-1,1) fp32, seeded)",
        "config": {"workload": "TBMM(B=500,N=26,M=72,K=26) + 2FCRelu(B=128,1128->128->64) + "
                               "MLP3(B=128,128->64->32->2) per step (BASELINE.json configs[1])",
                   "global_batch": {"tbmm": 500 * world, "fc": 128 * world}, "parallelism": f"dp{world}",
                   "l2": f"{nsets} rotating input+weight sets ({nsets * set_bytes / 2**20:.0f} MiB > 2x L2)",
                   "graphs": "one CUDA graph per input set (3 kernel launches)",
                   "flops_per_step": int(flops_step)},
        "e2e": {"value": round(e2e_value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "us_per_step": round(e2e_t / ke * 1e6, 2)},
        "gpu_launches": 3 * args.steps,
        "roofline": roofline,
        "step_ops": roofline_ops,
        "clocks": clk.summary(),
        "device": device_info(local),
    }
    if not args.no_ops:
        line["ops"] = paper_op_table(ee, torch, dev, stream, peaks)
    if world == 1 and not args.no_cpu_baseline:
        v, dt, info = cpu_reference_sample()
        line["cpu_baseline"] = {"value": round(v, 4), "unit": "GFLOP/s", **info}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def paper_op_table(ee, torch, dev, stream, peaks):
    """µs/call (device, L2-cold where the working set allows rotation) and the
    paper's protocol (p50 of synchronised calls incl. host overhead,
    PAPER.md:1570-1585) for every paper operator at its paper shape."""
    out = {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    for name, label, shapes, seeded in PAPER_OPS:
        try:
            big = name in ("2LUT", "gconv")
            one = OpInstance(ee, torch, name, shapes, seeded, 1, dev, 3)
            nsets = 1 if big else max(2, int(np.ceil(2 * L2_BYTES / max(1, one.set_bytes()))))
            nsets = min(nsets, 64)
            o = one if nsets == 1 else OpInstance(ee, torch, name, shapes, seeded, nsets, dev, 3)
            with torch.cuda.stream(stream):
                for i in range(3):
                    o.run(i)
                torch.cuda.synchronize()
                # one graph: `per` launches rotating over the input sets
                per = max(nsets, 8 if big else 32)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for i in range(per):
                        o.run(i)
                for i in range(2):
                    g.replay()
                reps = 3 if name == "gconv" else 10
                t = time_device(torch, lambda i: g.replay(), reps, stream) / (reps * per)
                # paper protocol: synchronised single calls incl. launch overhead
                lat = []
                for i in range(100 if name == "gconv" else 300):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    o.run(i)
                    torch.cuda.synchronize()
                    lat.append(time.perf_counter() - t0)
            lat.sort()
            out[label] = {"us": round(t * 1e6, 3), "gflops": round(o.flops / t / 1e9, 1),
                          "hbm_gbs": round(o.bytes / t / 1e9, 1), "hbm_frac": round(o.bytes / t / 1e9 / hbm, 4),
                          "us_p0_p50_p90_sync": [round(lat[0] * 1e6, 1), round(lat[len(lat) // 2] * 1e6, 1),
                                                 round(lat[int(len(lat) * 0.9)] * 1e6, 1)],
                          "l2": "cold (rotated)" if nsets > 1 else "warm (working set > L2)" if big else "warm",
                          "kernel": o.kernel}
            del o, one
            torch.cuda.empty_cache()
        except Exception as e:  # report, don't hide
            out[label] = {"error": f"{type(e).__name__}: {e}"}
    return out


if __name__ == "__main__":
    main()
