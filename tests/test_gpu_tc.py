"""GPU parity of the tensor-core (tcgen05 TF32 / 3xTF32) variants. These
variants are not FFMA-exact: a tensor-core reduction cannot reproduce the
reference interpreter's per-step fp32 chain (interpreter.cc:218-233), so the
bar is a stated tolerance, on maxRelError
(tensor_data.cc:221-234, denominator max(|ref|, 1)):

  1. against the tensor-core emulation (tests/tc_emulate.py: the operands
     rounded exactly as the kernels round them, products summed in fp64):
       <= tol_emu(K) = r * K * 2^-24 * max(1, max|a| max|b|), r = the MMAs
          issued into the accumulator per k (tf32: 1, 3xtf32: 3)
     — only the fp32 accumulator's rounding separates the two, so a kernel
     that dropped one 32-deep k-block (~0.1 relative) fails by ~1000x;
  2. against the oracle (the reference's own fp32 chain), the operand-
     rounding bound, a sanity check on the emulation itself:
       3xtf32:  <= 1e-5 + K * 2^-23        tf32:  <= K * 2^-11

Every case records its measured errors next to the bounds
(gpurun_out/tc_errors.jsonl when run on the GPU box).
"""
import json
import os

import numpy as np
import pytest

import tc_emulate as emu
from conftest import max_rel
from oracle_lib import Oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def tol(math, K, scale=1.0):
    """scale = max|a| * max|b| of the contraction's operands (1 for U[-1,1) inputs)."""
    return (1e-5 + K * 2.0 ** -23 if math == "3xtf32" else K * 2.0 ** -11) * max(1.0, scale)


def opscale(a, b):
    return float(np.max(np.abs(a))) * float(np.max(np.abs(b)))


def record(name, math, K, err, exact_err, oracle_exact_err, emu_err=None, emu_bound=None):
    d = os.path.join(ROOT, "gpurun_out")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "tc_errors.jsonl"), "a") as f:
        f.write(json.dumps({"case": name, "math": math, "K": K, "max_rel_vs_oracle": err, "bound": tol(math, K),
                            "max_rel_vs_emulation": emu_err, "emulation_bound": emu_bound,
                            "max_rel_vs_fp64": exact_err, "oracle_max_rel_vs_fp64": oracle_exact_err}) + "\n")


def check_emu(name, math, K, got, ref_emu, scale=1.0):
    """The tight bar: got vs the tensor-core emulation."""
    e = max_rel(ref_emu, got)
    b = emu.tol_emu(K, scale, math)
    assert e <= b, f"{name} {math}: maxRel vs emulation {e:.3g} > {b:.3g}"
    return e, b


@pytest.fixture(scope="module")
def env():
    assert torch.cuda.is_available()
    from paper_1802_04730_b200 import ExecutionEngine
    return ExecutionEngine(), Oracle()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run(ee, name, params, outs, math, options=None):
    p = [dev(x) for x in params]
    o = [dev(x) for x in outs]
    h = ee.compile(name, p, o, options, math=math)
    ee.run(h, p, o)
    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in o], ee.describe(h)


def gemm64(A, B):
    return A.astype(np.float64) @ B.astype(np.float64).T


GEMM_CASES = [
    ("tmm", (128, 256, 32)),
    ("tmm", (128, 1024, 1024)),
    ("tmm", (200, 72, 64)),
    ("tmm", (77, 300, 44)),
    ("C3", (128, 1000, 1024)),
    ("C3", (5, 33, 20)),
]


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("name,shape", GEMM_CASES)
def test_gemm_tc(env, name, shape, math):
    ee, orc = env
    M, N, K = shape
    rng = orc.rng(11 + M + N + K)
    A, B = rng.f32((M, K)), rng.f32((N, K))
    if name == "C3":
        cin = rng.f32((M, N))
        ref = orc.c3(A, B, cin)
        exact = cin.astype(np.float64) + gemm64(A, B)
        (got,), desc = run(ee, "C3", [A, B], [cin], math)
    else:
        ref = orc.tmm(A, B)
        exact = gemm64(A, B)
        (got,), desc = run(ee, "tmm", [A, B], [np.zeros((M, N), np.float32)], math)
    assert desc["math"] == math and "tcgen05" in desc["kernel"]
    ref_emu = emu.gemm_nt(A, B, math) + (cin.astype(np.float64) if name == "C3" else 0.0)
    ee_, eb = check_emu(f"{name} {shape}", math, K, got, ref_emu)
    err = max_rel(ref, got)
    record(f"{name} {M}x{N}x{K}", math, K, err, max_rel(exact, got), max_rel(exact, ref), ee_, eb)
    assert err <= tol(math, K), f"{name} {shape} {math}: maxRel {err:.3g} > {tol(math, K):.3g}"


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("shape", [(500, 26, 72, 26), (7, 26, 72, 26), (3, 40, 36, 130)])
def test_tbmm_tc(env, shape, math):
    ee, orc = env
    Bt, N, M, K = shape  # tbmm.tc: X[B][N][M], Y[B][K][M] -> Z[B][N][K]
    rng = orc.rng(5 + Bt)
    X, Y = rng.f32((Bt, N, M)), rng.f32((Bt, K, M))
    ref = orc.tbmm(X, Y)
    exact = np.einsum("bnm,bkm->bnk", X.astype(np.float64), Y.astype(np.float64))
    (got,), desc = run(ee, "tbmm", [X, Y], [np.zeros((Bt, N, K), np.float32)], math)
    ee_, eb = check_emu(f"tbmm {shape}", math, M, got, emu.gemm_nt(X, Y, math))
    err = max_rel(ref, got)
    record(f"tbmm {shape}", math, M, err, max_rel(exact, got), max_rel(exact, ref), ee_, eb)
    assert err <= tol(math, M)


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("shape", [(128, 1128, 128, 64), (77, 300, 96, 40), (16, 64, 32, 2)])
def test_fc2_fused_tc(env, math, shape):
    """The fused two-layer tcgen05 kernel (tile_sizes[2] == 2: layer 1 split-K
    over a cluster, its reduced rows bulk-copied into rank 0, layer 2 there):
    both layers within the emulation bound at the paper shape and ragged ones
    (rows < 128, layer-2 width not a multiple of 16, a short last k-block)."""
    ee, orc = env
    B, K, N1, N2 = shape
    rng = orc.rng(7 + B)
    I, W1, B1 = rng.f32((B, K)), rng.f32((N1, K)), rng.f32((N1,))
    W2, B2 = rng.f32((N2, N1)), rng.f32((N2,))
    opts = {"block_shape": [1, 1, 1], "fusion_strategy": "max", "rng_seed": 0, "shared_memory_budget": 49152,
            "thread_shape": [256, 1, 1], "tile_sizes": [128, 1, 2], "unroll_copy_shared": False,
            "unroll_factor": 1, "use_private": False, "use_shared": True}
    (h1, h2), desc = run(ee, "2FCRelu", [I, W1, B1, W2, B2], [np.zeros((B, N1), np.float32),
                                                              np.zeros((B, N2), np.float32)], math, opts)
    assert "fused 2-layer" in desc["kernel"]
    ee1, eb1 = check_emu(f"fc2 {shape} layer 1", math, K, h1, emu.fc_relu(I, W1, B1, math))
    ee2, eb2 = check_emu(f"fc2 {shape} layer 2", math, N1, h2, emu.fc_relu(h1, W2, B2, math), opscale(h1, W2))
    record(f"fc2 fused {shape} layer 2", math, N1, max_rel(orc.fc_relu(h1, W2, B2), h2), None, None, ee2, eb2)


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
def test_fc_chains_tc(env, math):
    ee, orc = env
    rng = orc.rng(99)
    I, W1, B1 = rng.f32((128, 1128)), rng.f32((128, 1128)), rng.f32((128,))
    W2, B2 = rng.f32((64, 128)), rng.f32((64,))
    o1 = orc.fc_relu(I, W1, B1)
    o2 = orc.fc_relu(o1, W2, B2)
    (g1,), desc = run(ee, "MLP1", [I, W1, B1], [np.zeros((128, 128), np.float32)], math)
    assert "tcgen05" in desc["kernel"]
    ee1, eb1 = check_emu("MLP1", math, 1128, g1, emu.fc_relu(I, W1, B1, math))
    e1 = max_rel(o1, g1)
    record("MLP1 128x1128->128", math, 1128, e1, None, None, ee1, eb1)
    assert e1 <= tol(math, 1128)
    (h1, h2), _ = run(ee, "2FCRelu", [I, W1, B1, W2, B2], [np.zeros((128, 128), np.float32),
                                                           np.zeros((128, 64), np.float32)], math)
    check_emu("2FCRelu layer 1", math, 1128, h1, emu.fc_relu(I, W1, B1, math))
    assert max_rel(o1, h1) <= tol(math, 1128)
    # layer 2 consumes the GPU's own layer-1 output: compare against the
    # oracle / emulation applied to that same input
    ref2 = orc.fc_relu(h1, W2, B2)
    ee2, eb2 = check_emu("2FCRelu layer 2", math, 128, h2, emu.fc_relu(h1, W2, B2, math), opscale(h1, W2))
    e2 = max_rel(ref2, h2)
    record("2FCRelu layer 2", math, 128, e2, None, None, ee2, eb2)
    assert e2 <= tol(math, 128, opscale(h1, W2))
    O1 = rng.f32((128, 128))
    M2, C2, M3, C3b, M4, C4 = (rng.f32((64, 128)), rng.f32((64,)), rng.f32((32, 64)), rng.f32((32,)),
                               rng.f32((2, 32)), rng.f32((2,)))
    (q1, q2, q3, q4), _ = run(ee, "MLP3", [O1, M2, C2, M3, C3b, M4, C4],
                              [O1, np.zeros((128, 64), np.float32), np.zeros((128, 32), np.float32),
                               np.zeros((128, 2), np.float32)], math)
    assert np.array_equal(q1, O1)  # pass-through return untouched
    for got, (inp, W, b, K) in zip((q2, q3, q4), ((O1, M2, C2, 128), (q2, M3, C3b, 64), (q3, M4, C4, 32))):
        ee_, eb = check_emu(f"MLP3 layer K={K}", math, K, got, emu.fc_relu(inp, W, b, math), opscale(inp, W))
        e = max_rel(orc.fc_relu(inp, W, b), got)
        record(f"MLP3 layer K={K}", math, K, e, None, None, ee_, eb)
        assert e <= tol(math, K, opscale(inp, W))


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("B,K1,N1,N2,N3", [(77, 128, 64, 32, 2), (200, 64, 96, 64, 8), (130, 32, 64, 32, 36)])
def test_fc_fused_tc_ragged(env, math, B, K1, N1, N2, N3):
    """The one-kernel tcgen05 FC chain at ragged shapes: batches that leave a
    partial 128-row CTA, layer widths whose TMA-stored returns end inside a
    32-column box (clipped by the tensor map) and a last layer narrower than
    a 16-byte row (lane stores)."""
    ee, orc = env
    rng = orc.rng(B + N1 + N3)
    O1 = rng.f32((B, K1))
    M2, C2, M3, C3b, M4, C4 = (rng.f32((N1, K1)), rng.f32((N1,)), rng.f32((N2, N1)), rng.f32((N2,)),
                               rng.f32((N3, N2)), rng.f32((N3,)))
    (q1, q2, q3, q4), desc = run(ee, "MLP3", [O1, M2, C2, M3, C3b, M4, C4],
                                 [O1, np.zeros((B, N1), np.float32), np.zeros((B, N2), np.float32),
                                  np.zeros((B, N3), np.float32)], math)
    assert "fused chain" in desc["kernel"]
    assert np.array_equal(q1, O1)
    for got, (inp, W, b, K) in zip((q2, q3, q4), ((O1, M2, C2, K1), (q2, M3, C3b, N1), (q3, M4, C4, N2))):
        ee_, eb = check_emu(f"fused chain {B}x{K1} layer K={K}", math, K, got, emu.fc_relu(inp, W, b, math),
                            opscale(inp, W))
        e = max_rel(orc.fc_relu(inp, W, b), got)
        record(f"fused chain {B}x{K1} layer K={K}", math, K, e, None, None, ee_, eb)
        assert e <= tol(math, K, opscale(inp, W))


def test_tc_explicit_plan_and_errors(env):
    from paper_1802_04730_b200 import TcError, options_baseline
    ee, orc = env
    rng = orc.rng(3)
    A, B = rng.f32((128, 256)), rng.f32((512, 256))
    ref = orc.tmm(A, B)
    for bn, sp in [(16, 1), (16, 4), (64, 4), (128, 8), (256, 16), (32, 2)]:
        opts = json.loads(options_baseline(0))
        opts.update({"tile_sizes": [128, bn, 32], "block_shape": [1, 1, sp], "thread_shape": [256, 1, 1],
                     "use_shared": True, "fusion_strategy": "min"})
        (got,), desc = run(ee, "tmm", [A, B], [np.zeros((128, 512), np.float32)], "3xtf32", opts)
        assert f"bn={bn} splits={sp}" in desc["kernel"]
        check_emu(f"tmm bn={bn} splits={sp}", "3xtf32", 256, got, emu.gemm_nt(A, B, "3xtf32"))
        assert max_rel(ref, got) <= tol("3xtf32", 256)
    # rows not a multiple of 16 bytes: no tensor-core kernel
    A2, B2 = rng.f32((16, 30)), rng.f32((16, 30))
    with pytest.raises(TcError) as ei:
        run(ee, "tmm", [A2, B2], [np.zeros((16, 16), np.float32)], "tf32")
    assert ei.value.kind == "MappingInvalid"
    # shapes the tensor-core 3-KRU does not take say so (D0 != D1)
    X = rng.f32((4, 16, 16, 16))
    Ws = [rng.f32((32, 16)), rng.f32((16, 16)), rng.f32((32, 16))]
    with pytest.raises(TcError) as ei:
        run(ee, "3KRU", Ws + [X], [np.zeros((4, 32, 16, 32), np.float32), np.zeros((4, 16, 16, 32), np.float32),
                                   np.zeros((4, 16, 16, 32), np.float32)], "tf32")
    assert ei.value.kind == "MappingInvalid"


GCONV_CASES = [  # (N, G, C, H, W, F, KH, KW, Mb)
    (2, 3, 16, 10, 10, 16, 3, 3, 16),
    (1, 2, 16, 58, 58, 16, 3, 3, 16),     # the paper shape's N=1, G=2 slice
    (3, 2, 8, 20, 36, 32, 3, 3, 4),       # 34-wide rows (VW=64), 8 channels, F=32
    (2, 1, 16, 12, 20, 16, 5, 5, 3),      # 5x5 taps, 16-wide rows (VW=32)
]


@pytest.mark.parametrize("variant", ["nhwc", "im2col", "shift"])
@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("case", GCONV_CASES)
def test_gconv_tc(env, case, math, variant):
    """variant: the on-chip im2col kernel, the NHWC-staging kernel
    (tile_sizes[2] == 2) or the shifted-halo kernel (tile_sizes[2] == 3)."""
    from paper_1802_04730_b200 import options_baseline
    ee, orc = env
    N, G, C, H, W, F, KH, KW, Mb = case
    rng = orc.rng(31 + H + F)
    I, W1, Bv = rng.f32((N, G, C, H, W)), rng.f32((G, F, C, KH, KW)), rng.f32((Mb,))
    ref = orc.gconv(I, W1, Bv)
    opts = json.loads(options_baseline(0))
    opts.update({"tile_sizes": [128, F, {"nhwc": 2, "im2col": 1, "shift": 3}[variant]],
                 "thread_shape": [512, 1, 1]})
    (got,), desc = run(ee, "gconv", [I, W1, Bv], [np.zeros(ref.shape, np.float32)], math, opts)
    assert "tcgen05" in desc["kernel"]
    assert {"nhwc": "NHWC", "im2col": "im2col", "shift": "shifted halo"}[variant] in desc["kernel"]
    K = C * KH * KW
    ref_emu = emu.gconv_points(I, W1, Bv, np.arange(got.size), math)
    ee_, eb = check_emu(f"gconv {case} {variant}", math, K + Mb, got.reshape(-1), ref_emu)
    err = max_rel(ref, got)
    record(f"gconv {case} {variant}", math, K, err, None, None, ee_, eb)
    assert err <= tol(math, K), f"gconv {case} {math}: maxRel {err:.3g} > {tol(math, K):.3g}"


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("case", [(1, 2, 8, 11, 13, 16, 3, 3, 2), (2, 1, 16, 9, 7, 32, 2, 2, 1)])
def test_gconv_tc_shift_odd_planes(env, case, math):
    """Shifted-halo kernel on planes with H*W % 4 != 0 (its 4-byte cp.async
    builders; the 4x4 vector builders need whole 16-byte pixel quads)."""
    from paper_1802_04730_b200 import options_baseline
    ee, orc = env
    N, G, C, H, W, F, KH, KW, Mb = case
    rng = orc.rng(7 + H * W)
    I, W1, Bv = rng.f32((N, G, C, H, W)), rng.f32((G, F, C, KH, KW)), rng.f32((Mb,))
    ref = orc.gconv(I, W1, Bv)
    opts = json.loads(options_baseline(0))
    opts.update({"tile_sizes": [128, F, 3], "thread_shape": [512, 1, 1]})
    (got,), desc = run(ee, "gconv", [I, W1, Bv], [np.zeros(ref.shape, np.float32)], math, opts)
    assert "shifted halo" in desc["kernel"]
    K = C * KH * KW
    ref_emu = emu.gconv_points(I, W1, Bv, np.arange(got.size), math)
    ee_, eb = check_emu(f"gconv {case} shift-odd", math, K + Mb, got.reshape(-1), ref_emu)
    err = max_rel(ref, got)
    record(f"gconv {case} shift-odd", math, K, err, None, None, ee_, eb)
    assert err <= tol(math, K), f"gconv {case} {math}: maxRel {err:.3g} > {tol(math, K):.3g}"


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("variant", [None, 3])
def test_gconv_tc_paper_shape_sampled(env, variant, math):
    """tcgen05 gconv at the BASELINE shape (32,32,16,16,58x58,3x3), 200k
    sampled points vs the emulation and the oracle (default plan, and the
    shifted-halo kernel explicitly), both math modes."""
    from paper_1802_04730_b200 import options_baseline
    ee, orc = env
    rng = orc.rng(11)
    I, W1, Bv = rng.f32((32, 32, 16, 58, 58)), rng.f32((32, 16, 16, 3, 3)), rng.f32((16,))
    opts = None
    if variant is not None:
        opts = json.loads(options_baseline(0))
        opts.update({"tile_sizes": [128, 16, variant], "thread_shape": [512, 1, 1]})
    (got,), desc = run(ee, "gconv", [I, W1, Bv], [np.zeros((32, 32, 16, 56, 56), np.float32)], math, opts)
    assert "tcgen05" in desc["kernel"]
    idx = np.random.default_rng(0).integers(0, got.size, 200_000)
    g = got.reshape(-1)[idx]
    ee_, eb = check_emu("gconv paper shape sampled", math, 144 + 16, g, emu.gconv_points(I, W1, Bv, idx, math))
    ref = orc.gconv_points(I, W1, Bv, idx)
    err = max_rel(ref, g)
    record(f"gconv paper shape sampled ({desc['kernel']})", math, 144, err, None, None, ee_, eb)
    assert err <= tol(math, 144)


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("shape", [(3, 32, 48), (2, 16, 16), (8, 32, 32)])  # (M, D0 = D1, D2)
def test_kru_tc(env, shape, math):
    """tcgen05 3-KRU (tc_kru.cu): three chained K = 16 contractions, each
    return within the stated bound for its depth in the chain (the K of every
    contraction feeding it), scaled by the operand magnitudes."""
    ee, orc = env
    M, D, D2 = shape
    rng = orc.rng(5 + M + D + D2)
    W0, W1, W2 = rng.f32((D, 16)), rng.f32((D, 16)), rng.f32((D2, 16))
    X = rng.f32((M, 16, 16, 16))
    Y, XW1, XW2 = orc.kru3(W0, W1, W2, X)
    outs = [np.zeros(Y.shape, np.float32), np.zeros(XW1.shape, np.float32), np.zeros(XW2.shape, np.float32)]
    (gY, gXW1, gXW2), desc = run(ee, "3KRU", [W0, W1, W2, X], outs, math)
    assert "tcgen05" in desc["kernel"] and "3-step" in desc["kernel"]
    # emulation stage by stage, each fed the GPU's own previous return (the
    # kernel's next A operand is exactly that fp32 accumulator value)
    e2 = emu.gemm_nt(X.reshape(-1, 16), W2, math).reshape(gXW2.shape)
    t = np.ascontiguousarray(np.transpose(gXW2, (0, 1, 3, 2)))            # [m,n0,d2,r1]
    e1 = np.transpose(emu.gemm_nt(t.reshape(-1, 16), W1, math).reshape(M, 16, D2, D), (0, 1, 3, 2))
    t = np.ascontiguousarray(np.transpose(gXW1, (0, 2, 3, 1)))            # [m,d1,d2,r0]
    e0 = np.transpose(emu.gemm_nt(t.reshape(-1, 16), W0, math).reshape(M, D, D2, D), (0, 3, 1, 2))
    for name, got, ref_e, K, scale in (("XW2", gXW2, e2, 16, opscale(X, W2)), ("XW1", gXW1, e1, 16, opscale(gXW2, W1)),
                                       ("Y", gY, e0, 16, opscale(gXW1, W0))):
        check_emu(f"3KRU {shape} {name}", math, K, got, ref_e, scale)
    for name, got, ref, K, scale in (("XW2", gXW2, XW2, 16, opscale(X, W2)),
                                     ("XW1", gXW1, XW1, 32, opscale(XW2, W1)),
                                     ("Y", gY, Y, 48, opscale(XW1, W0))):
        err = max_rel(ref, got)
        record(f"3KRU {shape} {name}", math, K, err, None, None)
        assert err <= tol(math, K, scale), f"3KRU {shape} {name} {math}: maxRel {err:.3g} > {tol(math, K, scale):.3g}"


@pytest.mark.parametrize("math", ["tf32", "3xtf32"])
def test_tc_tuner_and_cache_replay(env, tmp_path, math):
    """The genetic tuner over the tcgen05 genes (tile N, K splits): every
    candidate is held to the mode's tolerance against the default plan, the
    cache records entries under the ' math=<mode>' target, and a later
    tensor-core compile replays the best plan while the FFMA compile of the
    same shapes does not see it."""
    import paper_1802_04730_b200 as tcb
    ee, orc = env
    tcb.cache_purge()
    rng = orc.rng(8)
    A, B, Cin = rng.f32((128, 1024)), rng.f32((1000, 1024)), rng.f32((128, 1000))
    ref = orc.c3(A, B, Cin)
    dA, dB = dev(A), dev(B)
    dC = dev(Cin)
    log = tmp_path / "tc_session.jsonl"
    best = ee.tune("C3", [dA, dB], [dC], population=10, generations=2, seed=3, timing_iters=3, math=math,
                   session_log=str(log))
    assert best["tile_sizes"][1] in (1, 16, 32, 64, 128, 256) and best["block_shape"][2] in (1, 2, 4, 8, 16)
    ents = tcb.cache_entries()
    assert len(ents) == 1 and ents[0]["target"].endswith(f" math={math}")
    costs = [json.loads(x)["best_cost"] for x in log.read_text().splitlines()]
    assert all(a >= b for a, b in zip(costs, costs[1:]))
    h = ee.compile("C3", [dA, dB], [dC], math=math)
    d = ee.describe(h)
    assert d["options_source"] == "cache" and d["options"] == best
    dC.copy_(torch.from_numpy(Cin))
    ee.run(h, [dA, dB], [dC])
    torch.cuda.synchronize()
    assert max_rel(ref, dC.cpu().numpy()) <= tol(math, 1024)
    assert ee.describe(ee.compile("C3", [dA, dB], [dC]))["options_source"] == "default"
    tcb.cache_purge()


def test_tmm_huge_paper_shape(env):
    """TMM at the paper's large shape (128, 4096, 16384),
    every math mode: the FFMA kernel bit-exact against the oracle on sampled
    rows, the tensor-core kernels within tol_emu of the emulation on sampled
    rows x columns."""
    ee, orc = env
    rng = orc.rng(1632)
    A, B = rng.f32((128, 16384)), rng.f32((4096, 16384))
    rows = np.array([0, 1, 37, 64, 101, 127])
    cols = np.sort(np.random.default_rng(1).choice(4096, 512, replace=False))
    cols[0], cols[-1] = 0, 4095
    dA, dB = dev(A), dev(B)
    ref_rows = orc.tmm(np.ascontiguousarray(A[rows]), B)                    # [6, 4096] fp32 chains
    for math in ("ffma", "tf32", "3xtf32"):
        dC = torch.zeros((128, 4096), device="cuda")
        h = ee.compile("tmm", [dA, dB], [dC], math=math)
        ee.run(h, [dA, dB], [dC])
        torch.cuda.synchronize()
        got = dC.cpu().numpy()[rows]
        kern = ee.describe(h)["kernel"]
        if math == "ffma":
            bad = int(np.sum(got.view(np.uint32) != ref_rows.view(np.uint32)))
            assert bad == 0, f"tmm 128x4096x16384 ffma ({kern}): {bad} sampled elements not bit-exact"
            record("tmm 128x4096x16384 sampled rows", math, 16384, max_rel(ref_rows, got), None, None, 0.0, 0.0)
            continue
        assert "tcgen05" in kern
        ref_e = emu.gemm_nt(A[rows], B[cols], math)
        ee_, eb = check_emu("tmm 128x4096x16384", math, 16384, got[:, cols], ref_e)
        err = max_rel(ref_rows[:, cols], got[:, cols])
        record(f"tmm 128x4096x16384 sampled ({kern})", math, 16384, err, None, None, ee_, eb)
        assert err <= tol(math, 16384)
