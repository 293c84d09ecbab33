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
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "µs/call and GFLOP/s per TC op at paper shapes (1/2/4/8 B200) vs roofline & CPU ref"
L2_BYTES = 126 * 1024 * 1024
STEP_WORKLOAD = "TBMM(B=500,N=26,M=72,K=26) + 2FCRelu(B=128,1128->128->64) + MLP3(B=128,128->64->32->2) per step"

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
    ("tmm", "tmm 128x4096x16384", [(128, 16384), (4096, 16384)], {}),
    ("tbmm", "tbmm 500,26,72,26", [(500, 26, 72), (500, 26, 72)], {}),
    ("MLP1", "MLP1 128x1128->128", [(128, 1128), (128, 1128), (128,)], {}),
    ("2FCRelu", "2FCRelu 128x1128->128->64", [(128, 1128), (128, 1128), (128,), (64, 128), (64,)], {}),
    ("MLP3", "MLP3 128->64->32->2", [(128, 128), (64, 128), (64,), (32, 64), (32,), (2, 32), (2,)],
     {0: (128, 128)}),
    ("C3", "C3 128x1024->1000", [(128, 1024), (1000, 1024)], {0: (128, 1000)}),
    ("3KRU", "3KRU M=256 16^3->32^3", [(32, 16), (32, 16), (32, 16), (256, 16, 16, 16)], {}),
    ("gconv", "gconv 32,32,16,16,58x58,3x3", [(32, 32, 16, 58, 58), (32, 16, 16, 3, 3), (16,)], {}),
    # the paper's four gconv columns (N,G,F,C,W,H) = (32,32,16,16,14,14), (32,32,32,32,7,7),
    # (32,32,4,4,56,56), (32,32,8,8,28,28): W,H are the outputs of 3x3 taps
    ("gconv", "gconv paper 32,32,16,16,14x14", [(32, 32, 16, 16, 16), (32, 16, 16, 3, 3), (16,)], {}),
    ("gconv", "gconv paper 32,32,32,32,7x7", [(32, 32, 32, 9, 9), (32, 32, 32, 3, 3), (32,)], {}),
    ("gconv", "gconv paper 32,32,4,4,56x56", [(32, 32, 4, 58, 58), (32, 4, 4, 3, 3), (4,)], {}),
    ("gconv", "gconv paper 32,32,8,8,28x28", [(32, 32, 8, 30, 30), (32, 8, 8, 3, 3), (8,)], {}),
    ("2LUT", "2LUT E=1e7,D=64,B=128,L=50",
     [(10_000_000, 64), (128, 50), (10_000_000, 64), (128, 50)], {}),
]
# tensor-core (tcgen05) variants of the contractions: (label of the exact op, math)
TC_OPS = [("tmm 128x1024x1024", "3xtf32"), ("tmm 128x1024x1024", "tf32"),
          ("tmm 128x4096x16384", "3xtf32"), ("tmm 128x4096x16384", "tf32"),
          ("C3 128x1024->1000", "3xtf32"), ("C3 128x1024->1000", "tf32"),
          ("tbmm 500,26,72,26", "3xtf32"), ("MLP1 128x1128->128", "3xtf32"),
          ("2FCRelu 128x1128->128->64", "3xtf32"), ("MLP3 128->64->32->2", "3xtf32"),
          ("gconv 32,32,16,16,58x58,3x3", "3xtf32"), ("gconv 32,32,16,16,58x58,3x3", "tf32"),
          ("3KRU M=256 16^3->32^3", "3xtf32"), ("3KRU M=256 16^3->32^3", "tf32"),
          ("gconv paper 32,32,16,16,14x14", "tf32"), ("gconv paper 32,32,32,32,7x7", "tf32")]
INT_PARAMS = {"2LUT": {1, 3}, "1LUT": {1}}
# Plans passed explicitly for the forked step (merged over each op's default
# options), measured over the step, not each op alone. Empty since the
# 9-rows-per-warp slab became the TBMM default: it is the best plan alone
# (6.7 us) and in the step (15.2 us; the 4-row slab that was the step plan:
# 16.0 us after the FC kernel changes, profiles/r02_slab_rows.txt). The
# library defaults are the standalone-best plans.
STEP_PLANS = {}


def step_set_bytes():
    """Bytes of one input+weight+output set of the step (all three ops), from
    the shapes alone: both arms derive the same `config` from it."""
    b = 0
    for name, shapes, seeded in STEP_OPS:
        b += sum(4 * int(np.prod(s)) for s in shapes)
    # outputs: TBMM Z, 2FCRelu O1+O2, MLP3 O1..O4
    b += 4 * (500 * 26 * 26 + 128 * 128 + 128 * 64 + 128 * 128 + 128 * 64 + 128 * 32 + 128 * 2)
    return b


def step_config(world):
    """The `config` object both arms print (same dict => same_config)."""
    nsets = max(2, int(np.ceil(2 * L2_BYTES / step_set_bytes())))
    return {"workload": STEP_WORKLOAD + " (BASELINE.json configs[1])",
            "global_batch": {"tbmm": 500 * world, "fc": 128 * world}, "parallelism": f"dp{world}",
            "l2": f"{nsets} rotating input+weight sets ({nsets * step_set_bytes() / 2**20:.0f} MiB > 2x L2)",
            "flops_per_step_per_rank": 90369280}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# --------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled DURING the timed
    region through NVML (a polling thread, ~1 ms period: the timed region is
    tens of ms, too short for `nvidia-smi -lms`)."""

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown")]

    def __init__(self, torch_dev):
        self.samples, self.max_mhz, self.reasons = [], None, set()
        self.h = None
        self.err = None
        try:
            import pynvml as N
            import torch
            N.nvmlInit()
            self.N = N
            pr = torch.cuda.get_device_properties(torch_dev)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            try:
                self.h = N.nvmlDeviceGetHandleByPciBusId_v2(bus.encode())
            except Exception:
                self.h = N.nvmlDeviceGetHandleByIndex(torch_dev.index or 0)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception as e:  # recorded, not hidden
            self.err = f"{type(e).__name__}: {e}"

    def _poll(self):
        N = self.N
        while not self.stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, const in self.REASONS:
                    if r & getattr(N, const, 0):
                        self.reasons.add(name)
            except Exception as e:
                self.err = f"{type(e).__name__}: {e}"
                return
            self.stop.wait(0.001)

    def __enter__(self):
        self.stop = threading.Event()
        if self.h is not None:
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.h is not None:
            self.t.join(timeout=5)

    def summary(self):
        out = {"sm_mhz": statistics.median(self.samples) if self.samples else None,
               "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
               "samples": len(self.samples), "source": "nvml, polled during the timed region"}
        if self.err:
            out["error"] = self.err
        return out


# ------------------------------------------------------------- workload
class OpInstance:
    """One TC op bound to device tensors (a rotating set of input copies)."""

    def __init__(self, ee, torch, name, pshapes, seeded, nsets, dev, seed, host_init=True, math="ffma", plan=None):
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
        opts = None
        if plan:
            opts = dict(ee.default_options(name, self.sets[0][0], self.sets[0][1]), **plan)
        self.handle = ee.compile(name, self.sets[0][0], self.sets[0][1], opts, math=math)
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


DOM_NOTES = {
    "2FCRelu": "Latency bound, not byte bound: every output is one sequential FFMA chain of 1128 + 128 dependent "
               "steps (chain_floor_us at 4 cycles a step); layer 1 runs two weight columns per thread at ~5.9 "
               "cycles a step (LDS.128 operand writeback of two CTAs per SM; one CTA per SM: ~5.0, "
               "profiles/r02_chain_probe2.txt) after ~1.1 us of prologue (copies issued by thread 0 first, "
               "landed ~2100 cycles after entry, profiles/r02_fc_early/; DESIGN.md section 8).",
    "tbmm": "500 batches of 26x26 outputs, 72-step chains, one wave of CTAs (slab kernel, 9 rows per warp). Phase "
            "trace (profiles/r02_slab_ws/trace_slab_c9_c4_c7.txt): its 8.84 MB are in by ~2.0 us (~4.6 TB/s; the "
            "cp.async issue itself stalls until then), then three 24-step chunks at ~0.9 us each, bound by the "
            "shared-memory pipe (a broadcast LDS.128 costs 2 wavefronts), stores done ~5.2 us (DESIGN.md "
            "sections 5 and 12).",
    "MLP3": "Three short dependent layers (128, 64, 32 steps): latency bound, see chain_floor_us.",
}


def chain_floor_us(op, fma_latency_cycles=4, mhz=1965.0):
    """Latency floor of an FFMA-exact operator: every output is one
    sequential chain of fused multiply-adds (the reference's reduction order),
    so the longest chain of dependent FMAs (summed over chained layers) times
    the FMA latency bounds the kernel from below."""
    steps = {"tbmm": 72, "2FCRelu": 1128 + 128, "MLP3": 128 + 64 + 32, "MLP1": 1128, "C3": 1024, "tmm": 32}
    return steps.get(op.name, 0) * fma_latency_cycles / mhz


def time_device(torch, fn, iters, stream, lead_in=None):
    """Device time of `iters` calls of fn(i) on `stream`, via CUDA events.
    lead_in: untimed work enqueued just before the start event (after the
    synchronize), so the GPU is already busy when the timed region opens and
    the host's submission of the timed graphs is not counted as device time
    (a 20-step graph launched onto an idle GPU exposed ~80 us of host submit
    latency, profiles/r02_final)."""
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if lead_in is not None:
        lead_in()
    s.record(stream)
    for i in range(iters):
        fn(i)
    e.record(stream)
    while not e.query():  # wait without holding the GIL: the clock sampler thread keeps polling
        time.sleep(0.0002)
    e.synchronize()
    return s.elapsed_time(e) * 1e-3  # seconds


# ----------------------------------------------------------- CPU baseline
class CpuStep:
    """The reference's own CPU implementation of the step — the interpreter
    backend::interpretReference (interpreter.cc:301-349) of the reference
    library compiled by oracle/Makefile (oracle/_ref) — over the step's work
    units: one TBMM batch (tbmm.tc), one 2FCRelu row, one MLP3 row, each a
    call of the reference through its public entry (parse + specialize +
    interpret). Units run on all host threads (the interpreter is reentrant,
    interpreter.h:78). A sample = the next `n` units of the step in
    round-robin order, so any number of samples covers the workload evenly.
    Without oracle/_ref, the C restatement (OpenMP) is timed instead
    ("port"). Test/bench infrastructure only."""

    def __init__(self, threads=None):
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_lib import Oracle, RefLib

        self.threads = threads or os.cpu_count() or 1
        orc = Oracle()
        rng = orc.rng(7)
        self.X, self.Y = rng.f32((500, 26, 72)), rng.f32((500, 26, 72))
        self.I, self.W1, self.B1 = rng.f32((128, 1128)), rng.f32((128, 1128)), rng.f32((128,))
        self.W2, self.B2 = rng.f32((64, 128)), rng.f32((64,))
        self.O1 = rng.f32((128, 128))
        self.M = [rng.f32((64, 128)), rng.f32((64,)), rng.f32((32, 64)), rng.f32((32,)),
                  rng.f32((2, 32)), rng.f32((2,))]
        self.units = [("tbmm", b) for b in range(500)]
        for r in range(128):
            self.units += [("2FCRelu", r), ("MLP3", r)]
        # interleave so any contiguous window mixes the three ops like the step
        self.units.sort(key=lambda u: (u[1] / (500 if u[0] == "tbmm" else 128), u[0]))
        self.flops = {"tbmm": 2.0 * 26 * 26 * 72, "2FCRelu": 2.0 * (128 * 1128 + 64 * 128),
                      "MLP3": 2.0 * (64 * 128 + 32 * 64 + 2 * 32)}
        self.cursor = 0
        self.orc = orc
        if RefLib.available():
            self.ref = RefLib()
            self.src = open(os.path.join(ROOT, "paper_1802_04730_b200", "tc", "ops.tc")).read()
            self.kind = "reference"
        else:
            self.ref = None
            self.kind = "port"
            orc.lib.orc_set_threads(self.threads)

    def _run_unit(self, u):
        op, i = u
        if op == "tbmm":
            self.ref.run(self.src, "tbmm", {"X": self.X[i:i + 1], "Y": self.Y[i:i + 1]}, ["Z"])
        elif op == "2FCRelu":
            self.ref.run(self.src, "2FCRelu", {"I": self.I[i:i + 1], "W1": self.W1, "B1": self.B1,
                                               "W2": self.W2, "B2": self.B2}, ["O1", "O2"])
        else:
            m = self.M
            self.ref.run(self.src, "MLP3", {"I": self.O1[i:i + 1], "W2": m[0], "B2": m[1], "W3": m[2],
                                            "B3": m[3], "W4": m[4], "B4": m[5], "O1": self.O1[i:i + 1]},
                         ["O2", "O3", "O4"])

    def _port(self, us):
        tb = [i for op, i in us if op == "tbmm"]
        fc = [i for op, i in us if op == "2FCRelu"]
        ml = [i for op, i in us if op == "MLP3"]
        if tb:
            self.orc.tbmm(self.X[tb], self.Y[tb])
        if fc:
            self.orc.fc_relu(self.orc.fc_relu(self.I[fc], self.W1, self.B1), self.W2, self.B2)
        if ml:
            m = self.M
            self.orc.mlp3(self.O1[ml], *m)

    def sample(self, n):
        """Run the next n units; returns (flops, seconds)."""
        import concurrent.futures as cf
        n = max(1, min(n, len(self.units)))
        us = [self.units[(self.cursor + k) % len(self.units)] for k in range(n)]
        self.cursor = (self.cursor + n) % len(self.units)
        t0 = time.perf_counter()
        if self.ref is not None:
            with cf.ThreadPoolExecutor(self.threads) as ex:
                list(ex.map(self._run_unit, us))
        else:
            self._port(us)
        dt = time.perf_counter() - t0
        return sum(self.flops[op] for op, _ in us), dt

    def units_for(self, seconds):
        """Units that take about `seconds` on all threads (calibrated)."""
        f, dt = self.sample(2 * self.threads)
        per = dt / (2 * self.threads)
        return max(1, int(seconds / per))

    def describe(self, n):
        return (f"{n} work units per sample (of the step's 756: 500 TBMM batches, 128 2FCRelu rows, "
                f"128 MLP3 rows), round-robin over the step, each a {self.kind} call")


def cpu_baseline(budget_s=15.0):
    """bench.py's cpu_baseline leg: ~budget_s of the reference's CPU path."""
    cs = CpuStep()
    n = cs.units_for(budget_s / 4)
    fl = tt = 0.0
    while tt < budget_s:
        f, dt = cs.sample(n)
        fl, tt = fl + f, tt + dt
    return fl / tt / 1e9, {"kind": cs.kind, "cores": cs.threads, "cpu_model": cpu_model(),
                           "sample": cs.describe(n) + f"; {tt:.1f} s timed"}


def cpu_baseline_port(budget_s=8.0):
    """The restated loop nests (oracle/oracle.c, OpenMP over the batch on all
    host threads: BASELINE.md section 3 path 2) over
    whole steps of the same workload: the honest compiled-CPU comparison
    beside the tree-walking interpreter."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Oracle
    orc = Oracle()
    threads = os.cpu_count() or 1
    orc.lib.orc_set_threads(threads)
    rng = orc.rng(7)
    X, Y = rng.f32((500, 26, 72)), rng.f32((500, 26, 72))
    I, W1, B1, W2, B2 = (rng.f32((128, 1128)), rng.f32((128, 1128)), rng.f32((128,)), rng.f32((64, 128)),
                         rng.f32((64,)))
    O1 = rng.f32((128, 128))
    M = [rng.f32((64, 128)), rng.f32((64,)), rng.f32((32, 64)), rng.f32((32,)), rng.f32((2, 32)), rng.f32((2,))]
    steps, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s or steps < 1:
        orc.tbmm(X, Y)
        orc.fc_relu(orc.fc_relu(I, W1, B1), W2, B2)
        orc.mlp3(O1, *M)
        steps += 1
    dt = time.perf_counter() - t0
    return 90369280 * steps / dt / 1e9, {"kind": "port", "cores": threads, "cpu_model": cpu_model(),
                                         "sample": f"{steps} whole steps of the restated C loops (OpenMP), "
                                                   f"{dt:.1f} s timed"}


def reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU implementation on the host
    cores, same metric/config; each step a bounded sample sized so the whole
    --steps/--warmup run takes about two minutes. Rank 0 only."""
    if rank != 0:
        return
    cs = CpuStep()
    per_step = min(10.0, 120.0 / (args.steps + args.warmup))
    n = cs.units_for(per_step)
    for _ in range(args.warmup):
        cs.sample(n)
    fl = tt = 0.0
    for _ in range(args.steps):
        f, dt = cs.sample(n)
        fl, tt = fl + f, tt + dt
    value = fl / tt / 1e9
    step_flops = 500 * cs.flops["tbmm"] + 128 * (cs.flops["2FCRelu"] + cs.flops["MLP3"])
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(step_flops / (value * 1e9) * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (U[-1,1) fp32, seeded)",
        "config": step_config(args.gpus),
        "note": "reference CPU interpreter on a bounded sample per step; ms_per_step is the full step's FLOPs "
                "at the measured rate",
        "cpu_baseline": {"value": round(value, 6), "unit": "GFLOP/s", "kind": cs.kind, "cores": cs.threads,
                         "sample": cs.describe(n), "cpu_model": cpu_model()},
        "e2e": {"value": round(value, 6), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- main arm
def _free_port():
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: re-exec this script under
    torch.distributed.run with N local ranks (one process per GPU), exactly
    as the driver launches it. Fails loudly when the box has fewer GPUs."""
    import subprocess

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and not args.allow_shared_gpu:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this box has {have}", file=sys.stderr)
        sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="tcb", choices=["tcb", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--serial-step", action="store_true", help="run the step's operators back to back on one stream")
    ap.add_argument("--no-ops", action="store_true", help="skip the per-op paper table")
    ap.add_argument("--profile-only", action="store_true", help="run a few steps, print nothing (ncu)")
    ap.add_argument("--allow-shared-gpu", action="store_true",
                    help="testing only: let N ranks share fewer GPUs (rank r on cuda:r %% count); NCCL is then "
                         "replaced by gloo for the gather")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)

    import torch
    import torch.distributed as dist

    from paper_1802_04730_b200 import ExecutionEngine, device_info, measure_peaks

    ndev = torch.cuda.device_count()
    if world > ndev and not args.allow_shared_gpu:
        print(f"bench.py: {world} ranks need {world} GPUs, this box has {ndev}", file=sys.stderr)
        sys.exit(2)
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    shared = world > ndev
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    peaks, peak_src = load_peaks()
    peaks = dict(peaks)
    mp = measure_peaks(local)  # measured now, this GPU
    peaks["ffma_tflops"] = round(mp["ffma_tflops"], 2)
    peaks["launch_floor_us"] = {k: round(v, 3) for k, v in mp["launch_floor_us"].items()}
    ee = ExecutionEngine()

    # rotating input sets larger than L2 (inputs AND weights rotate)
    nsets = max(2, int(np.ceil(2 * L2_BYTES / step_set_bytes())))
    ops = [OpInstance(ee, torch, n, s, sd, nsets, dev, 1 + i + 100 * rank, plan=STEP_PLANS.get(n)) for i, (n, s, sd)
           in enumerate(STEP_OPS)]
    set_bytes = sum(o.set_bytes() for o in ops)
    flops_step = sum(o.flops for o in ops)
    stream = torch.cuda.Stream(device=dev)
    # the step's three operators are independent: inside the graph they fork
    # onto their own streams and join back (concurrent kernels share the SMs)
    side = [torch.cuda.Stream(device=dev) for _ in ops]

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if not shared else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with torch.cuda.stream(stream):
        def fork_join(i, body):
            if args.serial_step:
                for o in ops:
                    body(o, i)
                return
            # every operator on its own side stream; the main stream only
            # forks and joins (profiles/r01_concurrency.txt)
            for sd in side:
                sd.wait_stream(stream)
            for o, sd in zip(ops, side):
                with torch.cuda.stream(sd):
                    body(o, i)
            for sd in side:
                stream.wait_stream(sd)

        def step(i):
            fork_join(i, lambda o, k: o.run(k))

        def graph_of(fn, idx):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for i in idx:
                    fn(i)
            return g

        for i in range(nsets):
            step(i)
        torch.cuda.synchronize()
        # K steps = (K // nsets) replays of a graph of all nsets steps + one
        # graph of the K % nsets remaining steps: every step sits inside a
        # graph beside its neighbours, whatever K is
        g_all = graph_of(step, range(nsets))
        full, rest = divmod(args.steps, nsets)
        g_rest = graph_of(step, range(rest)) if rest else None
        schedule = [g_all] * full + ([g_rest] if g_rest else [])
        for i in range(-(-args.warmup // nsets)):  # >= W warm-up steps
            g_all.replay()
        if g_rest:
            g_rest.replay()
        torch.cuda.synchronize()
        if args.profile_only:
            for g in schedule:
                g.replay()
            torch.cuda.synchronize()
            return

        # ---- timed region: K steps, barrier + sync both sides, max over ranks
        barrier()
        torch.cuda.synchronize()
        with ClockSampler(dev) as clk:  # (polls through the lead-in too: the GPU is under load throughout)
            lead = None if os.environ.get("TCB_BENCH_NO_LEADIN") else (lambda: g_all.replay())
            el = time_device(torch, lambda i: schedule[i].replay(), len(schedule), stream, lead_in=lead)
        torch.cuda.synchronize()
        # the timed region is K steps of ~16 us: too short for more than a
        # sample or two of a ~1 ms NVML poll, so the same step graph keeps
        # the GPU under the same load for ~30 ms right after it, polled too
        # (reported beside the timed region's own samples as `window`)
        with ClockSampler(dev) as clk_win:
            t_win = time.perf_counter()
            while time.perf_counter() - t_win < 0.03:
                for _ in range(20):
                    g_all.replay()
                torch.cuda.synchronize()
            win_ms = (time.perf_counter() - t_win) * 1e3
        barrier()
        el = max_over_ranks(el)
        value = world * flops_step * args.steps / el / 1e9
        ms_step = el / args.steps * 1e3

        # ---- N > 1: strong scaling: ONE global step (TBMM
        # B=500, FC B=128) split over the ranks through tcb_run_shard
        # (500 -> 250 / 125 / 63x4+62x4, 128 -> 64 / 32 / 16), compute only and
        # compute + the all-gather of every output slice (NCCL)
        strong = None
        if world > 1:
            from paper_1802_04730_b200.shard import BATCH_DIMS

            def shard_body(o, k):
                ps, os_ = o.sets[k % nsets]
                ee.run_shard(o.handle, ps, os_, rank, world, check_errors=False)

            def sstep(i):
                fork_join(i, shard_body)

            # gather buffers: every batched return, padded to the largest slice
            gat = []
            for o in ops:
                lo, hi, n = ee.shard_range(o.handle, rank, world)
                mx = ee.shard_range(o.handle, 0, world)[1]
                for ri in sorted(BATCH_DIMS[o.name][1]):
                    if o.name == "MLP3" and ri == 0:
                        continue  # O1 is a read-only pass-through input
                    t = o.sets[0][1][ri]
                    pad = torch.zeros((mx,) + tuple(t.shape[1:]), device=dev)
                    allb = torch.empty((world * mx,) + tuple(t.shape[1:]), device=dev)
                    gat.append((o, ri, lo, hi, pad, allb))

            def gather(i):
                for o, ri, lo, hi, pad, allb in gat:
                    pad[: hi - lo].copy_(o.sets[i % nsets][1][ri][lo:hi])
                    if shared:
                        torch.cuda.current_stream().synchronize()
                        parts = list(allb.cpu().chunk(world))
                        dist.all_gather(parts, pad.cpu())
                    else:
                        dist.all_gather_into_tensor(allb, pad)

            for i in range(3):
                sstep(i)
                gather(i)
            torch.cuda.synchronize()
            gs_all = graph_of(sstep, range(nsets))
            for _ in range(3):
                gs_all.replay()
            torch.cuda.synchronize()
            reps = max(2, args.steps // nsets)
            barrier()
            ec = max_over_ranks(time_device(torch, lambda i: gs_all.replay(), reps, stream))
            kg = max(10, min(200, args.steps // 10))
            barrier()

            def step_gather(i):
                sstep(i)
                gather(i)

            eg = max_over_ranks(time_device(torch, step_gather, kg, stream))
            strong = {"split": {o.name: [list(ee.shard_range(o.handle, r, world)[:2]) for r in range(world)]
                                for o in ops},
                      "ms_per_step_compute": round(ec / (reps * nsets) * 1e3, 5),
                      "value_compute": round(flops_step * reps * nsets / ec / 1e9, 3),
                      "ms_per_step_with_allgather": round(eg / kg * 1e3, 5),
                      "value_with_allgather": round(flops_step * kg / eg / 1e9, 3), "unit": "GFLOP/s",
                      "gathered_bytes_per_rank": int(sum(p.numel() * 4 for *_, p, _ in gat)),
                      "collective": ("gloo (shared GPU, testing)" if shared else
                                     "NCCL all_gather_into_tensor per output slice, after every step"),
                      "timing": "compute: CUDA graph of %d steps (tcb_run_shard per op, forked), max over "
                                "ranks; with_allgather: %d eager steps incl. the gathers" % (nsets, kg)}

        # ---- per-op device time inside the step (same stream, L2-rotated):
        # one graph launches the op on every rotating input set back to back
        per_op = []
        for o in ops:
            g = graph_of(lambda i: o.run(i), range(nsets))
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
            plan = STEP_PLANS.get(o.name)
            hh = ee.compile(o.name, hp, ho, dict(ee.default_options(o.name, hp, ho), **plan) if plan else None)
            host.append((hh, hp, ho))
            h2d += sum(x.numel() * 4 for x in hp) + sum(x.numel() * 4 for i, x in enumerate(ho) if i in o.inout)
            d2h += sum(x.numel() * 4 for x in ho)

        # the three independent calls are enqueued asynchronously
        # (TCB_RUN_ASYNC) on three streams from one host thread, then the
        # step waits for all three: their copies and kernels overlap. Each
        # call moves its small pinned tensors in one segment-copy launch
        # (DESIGN.md §8).
        e2e_streams = [torch.cuda.Stream(device=dev) for _ in host]
        prepared = [ee.prepare(hh, hp, ho) for hh, hp, ho in host]

        def e2e_step(i):
            if args.serial_step:
                for pr, st in zip(prepared, e2e_streams):
                    pr.run(stream=st.cuda_stream)
                return
            for pr, st in zip(prepared, e2e_streams):
                pr.run(stream=st.cuda_stream, sync=False)
            for st in e2e_streams:
                st.synchronize()

        # untimed warm-up: the first host calls run slow (pinned-page and IOMMU
        # mappings warming up), ~0.3 s
        for i in range(max(args.warmup, 1000)):
            e2e_step(i)
        # host wall clock (each step ends with its outputs on the host), in 5
        # blocks of kb steps; the median block is reported
        kb = max(4, args.steps // 20)
        ke = 5 * kb
        blocks = []
        barrier()
        for b in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(kb):
                e2e_step(b * kb + i)
            torch.cuda.synchronize()
            blocks.append(time.perf_counter() - t0)
        # pipelined: the same calls, but consecutive steps alternate between
        # two stream sets and the host waits once per block (each handle
        # alternates between two device staging sets, so step i+1's inputs
        # cross PCIe while step i computes and returns): every step still
        # moves its inputs H2D and its results D2H inside the timed region
        e2e_streams2 = [e2e_streams, [torch.cuda.Stream(device=dev) for _ in host]]

        kbp = 16  # steps per pipelined block (the host waits at its end)

        def e2e_block():
            for i in range(kbp):
                for pr, st in zip(prepared, e2e_streams2[i % 2]):
                    pr.run(stream=st.cuda_stream, sync=False)
            for sset in e2e_streams2:
                for st in sset:
                    st.synchronize()

        for i in range(20):
            e2e_block()
        pblocks = []
        barrier()
        for b in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_block()
            torch.cuda.synchronize()
            pblocks.append(time.perf_counter() - t0)
        # per-step seconds of each timing (median block), max over ranks
        us_sync = max_over_ranks(sorted(blocks)[2] / kb)
        us_pipe = max_over_ranks(sorted(pblocks)[2] / kbp)
        e2e_step_s = min(us_sync, us_pipe)
        e2e_value = world * flops_step / e2e_step_s / 1e9

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
    traffic = None
    try:  # committed ncu --set full capture of the same kernel
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)["per_launch"].get(dom.name, {})
            if tj.get("describe") in (None, dom.kernel):  # the capture is of this plan
                traffic = tj.get("dram_bytes")
    except Exception:
        traffic = None
    roofline = {"bound": "hbm", "kernel": f"{dom.name}: {dom.kernel}", "achieved": round(achieved, 1),
                "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                "traffic": int(traffic) if traffic else None,
                "traffic_source": "profiles/ncu_traffic.json (dram__bytes_read+write per launch, ncu --set full)",
                "algorithmic_bytes": int(dom.bytes), "launch_us": round(dom_t * 1e6, 3),
                "share_of_step": round(dom_t / step_dev, 3), "peak_source": peak_src,
                "note": "FFMA-exact fp32 kernels: no tensor-core roofline applies; HBM roofline over the "
                        "kernel's algorithmic bytes (inputs once, outputs once). chain_floor_frac = the "
                        "latency floor of its longest dependent FFMA chain / its time. " + DOM_NOTES.get(dom.name, ""),
                "chain_floor_us": round(chain_floor_us(dom), 3),
                "chain_floor_frac": round(chain_floor_us(dom) / (dom_t * 1e6), 4),
                # every kernel of the step on both bounds (the dominant one above)
                "by_kernel": {o.name: {"kernel": o.kernel, "launch_us": round(t * 1e6, 3),
                                       "hbm_achieved_gbs": round(o.bytes / t / 1e9, 1),
                                       "hbm_frac": round(o.bytes / t / 1e9 / hbm_peak, 4),
                                       "chain_floor_us": round(chain_floor_us(o), 3),
                                       "chain_floor_frac": round(chain_floor_us(o) / (t * 1e6), 4)}
                              for o, t in per_op}}
    roofline_ops = {
        o.name: {"us": round(t * 1e6, 3), "gflops": round(o.flops / t / 1e9, 1),
                 "hbm_gbs": round(o.bytes / t / 1e9, 1), "hbm_frac": round(o.bytes / t / 1e9 / hbm_peak, 4),
                 "ffma_frac": round(o.flops / t / 1e12 / peaks["ffma_tflops"], 4),
                 "chain_floor_us": round(chain_floor_us(o), 3),
                 "share": round(t / step_dev, 3), "kernel": o.kernel} for o, t in per_op}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (U[-1,1) fp32, seeded)",
        "config": step_config(world),
        "timing": {"graphs": "K // %d replays of one CUDA graph of all %d input sets' steps + one graph of the "
                             "K %% %d remaining steps (3 kernel launches per step); an untimed %d-step graph "
                             "replay leads into the start event" % (nsets, nsets, nsets, nsets) + (
                       ", operators serialised on one stream" if args.serial_step else
                       ", the 3 independent operators forked onto 3 streams and joined"),
                   "set_bytes": int(set_bytes), "nsets": nsets,
                   "step_plans": STEP_PLANS},
        "e2e": {"value": round(e2e_value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "us_per_step": round(e2e_step_s * 1e6, 2),
                "timing": "host wall clock, the faster of two timings of the same calls (median of 5 blocks "
                          "each): 'pipelined' = blocks of %d steps, each step the 3 tcb_run calls with pinned host "
                          "buffers (H2D + kernel + D2H) enqueued async, consecutive steps on alternating stream "
                          "sets, one host wait per block; 'sync_per_step' = blocks of %d steps, the host waits for "
                          "all 3 calls after every step" % (kbp, kb),
                "us_per_step_pipelined": round(us_pipe * 1e6, 2),
                "us_per_step_sync_per_step": round(us_sync * 1e6, 2),
                "blocks_us_per_step_sync": [round(x / kb * 1e6, 2) for x in blocks],
                "blocks_us_per_step_pipelined": [round(x / kbp * 1e6, 2) for x in pblocks]},
        "gpu_launches": 3 * args.steps,
        "strong": strong,
        "roofline": roofline,
        "step_ops": roofline_ops,
        "clocks": dict(clk.summary(), window=dict(clk_win.summary(), ms=round(win_ms, 1),
                                                    sm_mhz_min=min(clk_win.samples) if clk_win.samples else None,
                                                    source="nvml, the same step graph replayed right after "
                                                           "the timed region")),
        "peaks": {"hbm_gbs": hbm_peak, "hbm_source": peak_src, "ffma_tflops": peaks["ffma_tflops"],
                  "ffma_source": "measured in this run (tcb_measure_peaks: fma.rn.f32 chains, all SMs)",
                  "launch_floor_us": peaks["launch_floor_us"],
                  "launch_floor_source": "empty kernels replayed back to back from a CUDA graph (CTAs x threads)"},
        "device": device_info(local),
    }
    if not args.no_ops:
        line["ops"] = paper_op_table(ee, torch, dev, stream, peaks)
        line["prod_model"] = prod_model_line(ee, torch, dev)
    if world == 1 and not args.no_cpu_baseline:
        v, info = cpu_baseline()
        line["cpu_baseline"] = {"value": round(v, 6), "unit": "GFLOP/s", **info}
        v, info = cpu_baseline_port()
        line["cpu_baseline_port"] = {"value": round(v, 6), "unit": "GFLOP/s", **info}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def prod_model_line(ee, torch, dev):
    """The production model chain (2LUT -> C3 -> concat ->
    MLP1 -> MLP3) at the paper's sizes, one CUDA graph per forward pass:
    device µs per forward (median of 5 blocks of 100 back-to-back replays) and the paper-protocol
    synchronised latency."""
    try:
        from paper_1802_04730_b200.prodmodel import PAPER_SIZES as S
        from paper_1802_04730_b200.prodmodel import ProductionModel
        g = torch.Generator(device=dev)
        g.manual_seed(21)
        r = lambda *sh: torch.rand(sh, generator=g, device=dev) * 2 - 1  # noqa: E731
        p = dict(LUT1=r(S["E1"], S["D"]), LUT2=r(S["E2"], S["D"]),
                 I1=torch.randint(0, S["E1"], (S["B"], S["L1"]), generator=g, device=dev, dtype=torch.int32),
                 I2=torch.randint(0, S["E2"], (S["B"], S["L2"]), generator=g, device=dev, dtype=torch.int32),
                 I3=r(S["B"], S["WX"]), W=r(S["WY"], S["WX"]), W1=r(S["N"], 2 * S["D"] + S["WY"]), B1=r(S["N"]),
                 W2=r(S["O"], S["N"]), B2=r(S["O"]), W3=r(S["P"], S["O"]), B3=r(S["P"]), W4=r(S["Q"], S["P"]),
                 B4=r(S["Q"]))
        m = ProductionModel(ee, p).capture()
        for _ in range(5):
            m.replay()
        m.check()
        for _ in range(50):
            m.replay()
        n, blocks = 100, []
        for _ in range(5):  # median of 5 blocks: graph replays are host-launched
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(m.stream)
            for _ in range(n):
                m.replay()
            e1.record(m.stream)
            e1.synchronize()
            blocks.append(e0.elapsed_time(e1) * 1e3 / n)
        us = sorted(blocks)[2]
        lat = []
        for _ in range(100):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            m.replay()
            m.stream.synchronize()
            lat.append(time.perf_counter() - t0)
        lat.sort()
        out = {"us_per_forward": round(us, 3), "blocks_us_per_forward": [round(b, 2) for b in blocks],
               "gflops": round(m.flops / us / 1e3, 1),
               "us_p0_p50_p90_sync": [round(lat[0] * 1e6, 1), round(lat[50] * 1e6, 1), round(lat[90] * 1e6, 1)],
               "kernels": m.kernels, "graph": "C3 (tmm def, from zeros) -> 2LUT -> concat -> MLP1 -> MLP3, one CUDA graph on one stream",
               "sizes": S}
        del m, p
        torch.cuda.empty_cache()
        return out
    except Exception as e:  # report, don't hide
        return {"error": f"{type(e).__name__}: {e}"}


# the paper's latency protocol from C++ through the C ABI (`tcb latency`,
# csrc/cli/tcb_main.cc): 1000 synchronised tcb_run calls on device tensors
CLI_SIZES = {
    "tmm 128x256x32": ("tmm", "M=128,N=256,K=32"),
    "tmm 128x1024x1024": ("tmm", "M=128,N=1024,K=1024"),
    "tbmm 500,26,72,26": ("tbmm", "B=500,N=26,M=72,K=26"),
    "MLP1 128x1128->128": ("MLP1", "B=128,M=1128,O=128,N=1128"),
    "2FCRelu 128x1128->128->64": ("2FCRelu", "B=128,M=1128,O=128,N=1128,P=64"),
    "MLP3 128->64->32->2": ("MLP3", "B=128,M=128,O=64,N=128,P=32,Q=2,O1__0=128,O1__1=128"),
    "C3 128x1024->1000": ("C3", "B=128,WX=1024,WY=1000"),
    "3KRU M=256 16^3->32^3": ("3KRU", "D0=32,N0=16,D1=32,N1=16,D2=32,N2=16,M=256"),
}


def capi_latency(label, math="ffma", iters=1000, dev=0):
    if label not in CLI_SIZES:
        return None
    import subprocess
    d, sizes = CLI_SIZES[label]
    cmd = [os.path.join(ROOT, "paper_1802_04730_b200", "bin", "tcb"), "latency",
           os.path.join(ROOT, "paper_1802_04730_b200", "tc", "ops.tc"), "--def", d, "--sizes", sizes,
           "--iters", str(iters), "--math", math]
    env = dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", str(dev)))
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=120, env=env)
        j = json.loads(r.stdout.strip().splitlines()[-1])
        return {"us_p0_p50_p90_p99": [j["us_p0"], j["us_p50"], j["us_p90"], j["us_p99"]],
                "host_enqueue_us": j["host_enqueue_us"], "iters": j["iters"],
                "protocol": "C++ (bin/tcb latency): tcb_run on device tensors + stream sync, host wall clock"}
    except Exception as e:  # report, don't hide
        return {"error": f"{type(e).__name__}: {e}"}


def paper_op_table(ee, torch, dev, stream, peaks):
    """µs/call (device, L2-cold where the working set allows rotation) and the
    paper's protocol (p50 of synchronised calls incl. host overhead,
    PAPER.md:1570-1585) for every paper operator at its paper shape."""
    out = {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    byl = {lab: (n, sh, sd) for n, lab, sh, sd in PAPER_OPS}
    todo = [(n, lab, sh, sd, "ffma") for n, lab, sh, sd in PAPER_OPS]
    todo += [(*byl[lab][:1], f"{lab} [{m}]", *byl[lab][1:], m) for lab, m in TC_OPS]
    for name, label, shapes, seeded, math in todo:
        try:
            big = name in ("2LUT", "gconv") or label.startswith(("tmm 128x4096x16384", "gconv"))
            one = OpInstance(ee, torch, name, shapes, seeded, 1, dev, 3, math=math)
            nsets = 1 if big else max(2, int(np.ceil(2 * L2_BYTES / max(1, one.set_bytes()))))
            nsets = min(nsets, 64)
            o = one if nsets == 1 else OpInstance(ee, torch, name, shapes, seeded, nsets, dev, 3, math=math)
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
                reps = 3 if big else 10
                t = time_device(torch, lambda i: g.replay(), reps, stream) / (reps * per)
                # paper protocol: synchronised single calls incl. launch overhead
                lat = []
                for i in range(50 if big else 300):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    o.run(i)
                    torch.cuda.synchronize()
                    lat.append(time.perf_counter() - t0)
            lat.sort()
            out[label] = {"us": round(t * 1e6, 3), "gflops": round(o.flops / t / 1e9, 1),
                          "hbm_gbs": round(o.bytes / t / 1e9, 1), "hbm_frac": round(o.bytes / t / 1e9 / hbm, 4),
                          "ffma_frac": round(o.flops / t / 1e12 / peaks["ffma_tflops"], 4),
                          "us_p0_p50_p90_sync": [round(lat[0] * 1e6, 1), round(lat[len(lat) // 2] * 1e6, 1),
                                                 round(lat[int(len(lat) * 0.9)] * 1e6, 1)],
                          "l2": "cold (rotated)" if nsets > 1 else "warm (working set > L2)" if big else "warm",
                          "kernel": o.kernel, "math": math}
            if math == "ffma" or label == "tmm 128x256x32":
                out[label]["capi_sync_latency"] = capi_latency(label, math)
            if math != "ffma":
                # tensor-pipe roofline: TF32 dense = half the measured bf16 dense peak; 3xTF32
                # issues three TF32 MMAs per useful multiply-add
                tf32_peak = float(peaks.get("bf16_tflops", 1590.0)) / 2
                mult = 3 if math == "3xtf32" else 1
                out[label]["tensor_frac"] = round(mult * o.flops / t / 1e12 / tf32_peak, 4)
                out[label]["tensor_peak_tflops"] = round(tf32_peak, 1)
            del o, one
            torch.cuda.empty_cache()
        except Exception as e:  # report, don't hide
            out[label] = {"error": f"{type(e).__name__}: {e}"}
    return out


if __name__ == "__main__":
    main()
