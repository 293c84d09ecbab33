"""The paper's production model (`prodModel`) as ONE
CUDA graph over the tc-b200 kernels:

    (C1, C2) = 2LUT(LUT1, I1, LUT2, I2)           # embeddings, B x D each
    C3       = C3(I3, W)                           # += onto zeros (a fresh return): run as the
                                                   # tmm def (zero-init chain, same bits, no memset)
    I        = concat(C1, C2, C3)                  # B x (2D + WY); not expressible in TC
    O1       = MLP1(I, W1, B1)
    O2..O4   = MLP3(O1, W2, B2, W3, B3, W4, B4)

At the paper's sizes (E=1e7, D=64, L=50, B=128, WX=1024, WY=1000) the concat
width is 64+64+1000 = 1128, MLP1's input (mlp1.tc). The paper's motivation
for fusing is launch overhead in this low-latency
regime; here every launch of the chain is captured once and replayed: C3
(from zeros, as the tmm def), 2LUT, concat, MLP1 and MLP3 on one stream
(`fork=True` puts C3 beside 2LUT on a side stream; see __init__).
Each operator is the FFMA-exact kernel of its TC definition, so the chain's
outputs are bit-identical to evaluating the defs one after another on the
reference interpreter (tests/test_prodmodel.py).
"""
from __future__ import annotations

import ctypes as C

from ._lib import check, lib

PAPER_SIZES = dict(B=128, E1=10_000_000, E2=10_000_000, D=64, L1=50, L2=50, WX=1024, WY=1000, N=128, O=64, P=32,
                   Q=2)


class ProductionModel:
    """Binds the chain to caller-owned device tensors and replays it as one graph.

    params: dict with LUT1, I1, LUT2, I2, I3, W, W1, B1, W2, B2, W3, B3, W4, B4
    (torch CUDA tensors, float32 except the int32 index tensors I1, I2).
    Outputs (allocated here): C1, C2, C3, I, O1, O2, O3, O4.
    """

    def __init__(self, ee, params: dict, math: str = "ffma", fork: bool = False):
        import torch
        self.torch, self.ee = torch, ee
        # fork=True puts C3 on a side stream beside 2LUT. Measured on B200 the
        # forked graph is bimodal per block of replays (41.5 or 67.6 us per
        # forward: C3's CTAs placed beside 2LUT's run slow); one stream is a
        # steady 41.0 us (profiles/r01_prodmodel_probe.txt), so it is the default
        self.fork = fork
        p = self.p = params
        dev = p["I3"].device
        B, D = p["I1"].shape[0], p["LUT1"].shape[1]
        WY = p["W"].shape[0]
        N, O, P, Q = p["W1"].shape[0], p["W2"].shape[0], p["W3"].shape[0], p["W4"].shape[0]
        z = lambda *s: torch.zeros(s, device=dev, dtype=torch.float32)  # noqa: E731
        self.out = dict(C1=z(B, D), C2=z(B, D), C3=z(B, WY), I=z(B, 2 * D + WY), O1=z(B, N), O2=z(B, O),
                        O3=z(B, P), O4=z(B, Q))
        o = self.out
        self.h_lut = ee.compile("2LUT", [p["LUT1"], p["I1"], p["LUT2"], p["I2"]], [o["C1"], o["C2"]])
        # C3 from zeros: the `tmm` def's chain starts from 0.0 exactly as C3's
        # `+=` onto a zeroed return does (fma(a, b, 0) == a*b), so the zero
        # fill drops out of the critical path with identical bits
        self.h_c3 = ee.compile("tmm", [p["I3"], p["W"]], [o["C3"]], math=math)
        self.h_mlp1 = ee.compile("MLP1", [o["I"], p["W1"], p["B1"]], [o["O1"]], math=math)
        self.h_mlp3 = ee.compile("MLP3", [o["O1"], p["W2"], p["B2"], p["W3"], p["B3"], p["W4"], p["B4"]],
                                 [o["O1"], o["O2"], o["O3"], o["O4"]], math=math)
        self.kernels = {k: ee.describe(h)["kernel"] for k, h in
                        (("2LUT", self.h_lut), ("C3", self.h_c3), ("MLP1", self.h_mlp1), ("MLP3", self.h_mlp3))}
        self.flops = sum(ee.describe(h)["flops"] for h in (self.h_lut, self.h_c3, self.h_mlp1, self.h_mlp3))
        self.graph = None
        self.stream = torch.cuda.Stream(device=dev)
        self.side = torch.cuda.Stream(device=dev)

    def _concat(self, stream):
        o = self.out
        srcs = (C.c_void_p * 3)(o["C1"].data_ptr(), o["C2"].data_ptr(), o["C3"].data_ptr())
        widths = (C.c_int64 * 3)(o["C1"].shape[1], o["C2"].shape[1], o["C3"].shape[1])
        check(lib.tcb_concat_cols(srcs, widths, 3, o["I"].shape[0], C.c_void_p(o["I"].data_ptr()),
                                  C.c_void_p(stream.cuda_stream)))

    def _enqueue(self, check_errors):
        """Every launch of one forward pass on self.stream (+ the side stream)."""
        torch, ee, p, o = self.torch, self.ee, self.p, self.out
        s = self.stream
        c3s = self.side if self.fork else s
        c3s.wait_stream(s)
        with torch.cuda.stream(c3s):  # C3 onto a fresh zero return (the tmm def: zero-init chain)
            ee.run(self.h_c3, [p["I3"], p["W"]], [o["C3"]], stream=c3s.cuda_stream, check_errors=False)
        ee.run(self.h_lut, [p["LUT1"], p["I1"], p["LUT2"], p["I2"]], [o["C1"], o["C2"]], stream=s.cuda_stream,
               check_errors=check_errors)
        if self.fork:
            s.wait_stream(self.side)
        self._concat(s)
        ee.run(self.h_mlp1, [o["I"], p["W1"], p["B1"]], [o["O1"]], stream=s.cuda_stream, check_errors=False)
        ee.run(self.h_mlp3, [o["O1"], p["W2"], p["B2"], p["W3"], p["B3"], p["W4"], p["B4"]],
               [o["O1"], o["O2"], o["O3"], o["O4"]], stream=s.cuda_stream, check_errors=False)

    def forward_eager(self):
        """One pass without the graph (launch by launch); checks LUT indices."""
        self._enqueue(check_errors=True)
        self.stream.synchronize()
        return self.out

    def capture(self):
        torch = self.torch
        with torch.cuda.stream(self.stream):
            self._enqueue(check_errors=False)  # warm-up (kernel attributes set outside capture)
            self.stream.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=self.stream):
                self._enqueue(check_errors=False)
        return self

    def replay(self):
        """One forward pass = one graph launch (enqueued on self.stream)."""
        if self.graph is None:
            self.capture()
        with self.torch.cuda.stream(self.stream):
            self.graph.replay()

    def check(self):
        """Raises TcError(IndexOutOfRange) if a 2LUT index escaped its table since the last check."""
        self.stream.synchronize()
        self.ee.check(self.h_lut)

