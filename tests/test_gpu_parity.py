"""GPU parity: the CUDA path, called through the C ABI, against the
reference's own outputs (golden FNV hashes / vectors) and the pinned C
restatement. Bar: bit-exact (the FFMA-exact kernels run the reference's
reduction chain in order); every comparison also reports maxRelError
(tensor_data.cc:221-234) so a double-rounding tie would show as <= 1e-5."""
import json
import os

import numpy as np
import pytest

from cases import PARAM_ORDER, RETURN_ORDER, case_inputs, oracle_outputs
from conftest import fnv_hex, max_rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

_G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
CASES = sorted(_G["cases"])
TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.init()


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_on_gpu(engine, d, ins, seeded, options=None, host=False):
    params = [ins[n] for n in PARAM_ORDER[d]]
    given = [seeded[r].shape if r in seeded else None for r in RETURN_ORDER[d]]
    shapes = engine.infer_output_tensor_info(d, params, given)
    outs_np = [np.array(seeded[r], copy=True) if r in seeded else np.zeros(s, np.float32)
               for r, s in zip(RETURN_ORDER[d], shapes)]
    if host:
        p, o = params, outs_np
    else:
        p, o = [to_dev(x) for x in params], [to_dev(x) for x in outs_np]
    h = engine.compile(d, p, o, options)
    engine.run(h, p, o)
    if not host:
        torch.cuda.synchronize()
        o = [t.cpu().numpy() for t in o]
    return dict(zip(RETURN_ORDER[d], o)), h


def assert_exact(oracle, name, k, got, ref_fnv, ref_arr=None):
    if fnv_hex(oracle, got) == ref_fnv:
        return
    msg = f"{name}:{k} not bit-exact"
    if ref_arr is not None:
        diff = int(np.sum(got.view(np.uint32) != ref_arr.view(np.uint32)))
        msg += f" ({diff}/{got.size} elements differ, maxRel={max_rel(ref_arr, got):.3g})"
    raise AssertionError(msg)


@pytest.mark.parametrize("name", CASES)
def test_golden_bit_exact(engine, oracle, golden, name):
    case, ins, seeded = case_inputs(oracle, golden, name)
    got, _ = run_on_gpu(engine, case["def"], ins, seeded)
    ref = oracle_outputs(oracle, case, ins, seeded)
    for k, rec in case["outputs"].items():
        assert list(got[k].shape) == rec["shape"]
        assert max_rel(ref[k], got[k]) <= TOL
        assert_exact(oracle, name, k, got[k], rec["fnv"], ref[k])


@pytest.mark.parametrize("name", ["tmm_small", "tbmm_small", "c3_small", "mlp1_ragged"])
def test_every_gemm_variant_identical(engine, oracle, golden, name):
    """All instantiated GEMM kernels (and the direct one) give the same bits."""
    from paper_1802_04730_b200 import TcError
    case, ins, seeded = case_inputs(oracle, golden, name)
    ref = oracle_outputs(oracle, case, ins, seeded)
    base = json.loads(
        '{"block_shape":[1,1,1],"fusion_strategy":"max","rng_seed":0,"shared_memory_budget":49152,'
        '"thread_shape":[1,1,1],"tile_sizes":[32,32,32],"unroll_copy_shared":false,"unroll_factor":1,'
        '"use_private":true,"use_shared":true}')
    variants = [(16, 16, 1, 1, 32), (16, 32, 1, 2, 32), (32, 16, 2, 1, 32), (32, 32, 2, 2, 32),
                (32, 64, 2, 4, 32), (64, 32, 4, 2, 32), (64, 64, 4, 4, 32), (32, 32, 4, 4, 32),
                (16, 32, 2, 2, 32), (32, 32, 2, 2, 64), (64, 64, 4, 4, 16), (16, 64, 2, 4, 32),
                (32, 32, 2, 4, 32), (16, 16, 2, 2, 32), (32, 64, 4, 4, 32)]
    ran = 0
    for v in variants + [None]:
        o = dict(base)
        if v is None:
            o["use_shared"] = False
            o["thread_shape"] = [96, 1, 1]
        else:
            tm, tn, rm, rn, tk = v
            o["tile_sizes"] = [tm, tn, tk]
            o["thread_shape"] = [tn // rn, tm // rm, 1]
        if case["def"] == "MLP1":
            o["fusion_strategy"] = "min"
        got, _ = run_on_gpu(engine, case["def"], ins, seeded, options=o)
        for k in case["outputs"]:
            assert_exact(oracle, f"{name}/{o['tile_sizes']}", k, got[k], case["outputs"][k]["fnv"], ref[k])
        ran += 1
    assert ran == len(variants) + 1


TMA_VARIANTS = [(32, 32, 4, 4, 1), (32, 32, 4, 2, 1), (32, 64, 4, 4, 1), (16, 32, 2, 4, 1), (32, 16, 4, 2, 1),
                (64, 32, 4, 4, 1), (32, 32, 2, 2, 1), (32, 32, 2, 2, 4), (32, 32, 4, 2, 4), (32, 16, 2, 2, 4),
                (32, 32, 2, 2, 2)]


@pytest.mark.parametrize("name", ["tmm_small", "tbmm_small", "c3_small", "mlp1_ragged", "c3_paper", "tmm_paper",
                                  "tbmm_paper"])
def test_tma_gemm_variants(engine, oracle, golden, name):
    """The TMA-fed exact GEMM (gemm_tma.cu, tile_sizes[2] == 3) at every
    instantiated tile, bit-exact against the reference's goldens: ragged
    M/N edges (TMA zero fill, masked stores), a partial last k stage
    (K % 32 != 0), batches, in/out C3. Operands whose rows are not 16-byte
    multiples (mlp1_ragged) fall back to the tiled kernel, same bits. mc > 1:
    the A tile multicast over a cluster along N (grids padded to whole
    clusters: tmm_small's 48 columns are 2 tiles of a 4-cluster)."""
    case, ins, seeded = case_inputs(oracle, golden, name)
    ref = oracle_outputs(oracle, case, ins, seeded)
    for tm, tn, rm, rn, mc in TMA_VARIANTS:
        o = {"block_shape": [1, mc, 1], "fusion_strategy": "min" if case["def"] == "MLP1" else "max", "rng_seed": 0,
             "shared_memory_budget": 49152, "thread_shape": [tn // rn, tm // rm, 1], "tile_sizes": [tm, tn, 3],
             "unroll_copy_shared": False, "unroll_factor": 1, "use_private": True, "use_shared": True}
        got, h = run_on_gpu(engine, case["def"], ins, seeded, options=o)
        for k in case["outputs"]:
            assert_exact(oracle, f"{name}/tma{tm}x{tn}r{rm}x{rn}mc{mc}", k, got[k], case["outputs"][k]["fnv"], ref[k])


@pytest.mark.parametrize("name", ["tbmm_small", "tbmm_paper"])
def test_batched_persistent_variants(engine, oracle, golden, name):
    """The persistent batched kernel (tile_sizes[2] == 1) at every micro-tile
    and several grid sizes (1 CTA walking every batch, ragged splits, more
    CTAs than batches) gives the reference's bits."""
    case, ins, seeded = case_inputs(oracle, golden, name)
    ref = oracle_outputs(oracle, case, ins, seeded)
    base = json.loads(
        '{"block_shape":[1,1,1],"fusion_strategy":"max","rng_seed":0,"shared_memory_budget":49152,'
        '"thread_shape":[256,1,1],"tile_sizes":[2,2,1],"unroll_copy_shared":false,"unroll_factor":1,'
        '"use_private":true,"use_shared":true}')
    for rm, rn in [(1, 1), (1, 2), (2, 1), (2, 2)]:
        for grid in [1, 3, 7, 296, 1000]:
            o = dict(base)
            o["tile_sizes"] = [rm, rn, 1]
            o["block_shape"] = [grid, 1, 1]
            got, h = run_on_gpu(engine, case["def"], ins, seeded, options=o)
            assert "batched" in engine.describe(h)["kernel"]
            for k in case["outputs"]:
                assert_exact(oracle, f"{name}/{rm}x{rn}/grid{grid}", k, got[k], case["outputs"][k]["fnv"], ref[k])



@pytest.mark.parametrize("shape", [(500, 26, 26, 72), (37, 13, 29, 44), (3, 28, 32, 8), (9, 61, 40, 144)])
def test_slab_variants(engine, oracle, shape):
    """The slab kernel (tile_sizes[2] == 2, one CTA per batch, A rows
    broadcast from shared memory) at 4 to 7, 9 and 13 output rows per warp;
    ragged rows, columns and a short last reduction chunk; bit-exact vs the
    oracle."""
    B, N, K, M = shape  # Z(b,n,k) += X(b,n,m) * Y(b,k,m)
    rng = np.random.default_rng(B * 7 + M)
    X = rng.uniform(-1, 1, (B, N, M)).astype(np.float32)
    Y = rng.uniform(-1, 1, (B, K, M)).astype(np.float32)
    ref = oracle.tbmm(X, Y)
    for ch, l1 in [(4, False), (5, False), (6, False), (7, False), (9, False), (13, False)]:
        o = {"block_shape": [1, 1, 1], "fusion_strategy": "max", "rng_seed": 0, "shared_memory_budget": 49152,
             "thread_shape": [32, 1, 1], "tile_sizes": [ch, 1, 2], "unroll_copy_shared": l1, "unroll_factor": 1,
             "use_private": True, "use_shared": True}
        got, h = run_on_gpu(engine, "tbmm", {"X": X, "Y": Y}, {}, options=o)
        assert "slab_c" in engine.describe(h)["kernel"]
        diff = int(np.sum(got["Z"].view(np.uint32) != ref.view(np.uint32)))
        assert diff == 0, f"tbmm {shape} slab c{ch} l1={l1}: {diff} elements differ"


@pytest.mark.parametrize("rows,cn,threads", [(1, 1, 64), (2, 2, 64), (4, 8, 64), (8, 8, 64), (8, 4, 256),
                                             (16, 8, 128), (3, 3, 96), (8, 16, 64), (4, 8, 32), (5, 8, 64),
                                             (2, 4, 32), (1, 2, 32)])
def test_fc_chain_cluster_variants(engine, oracle, golden, rows, cn, threads):
    """Cluster sizes 1..16 (16 = non-portable), ragged rows and column splits.
    Blocks of half a layer's chains run column pairs per thread (planFc's
    `pair`: (4, 8, 32), (5, 8, 64), (8, 8, 64), ...), including a second
    column past a ragged layer's width.
    Combinations whose weight slices exceed shared memory must be rejected
    with MappingInvalid (never silently run)."""
    from paper_1802_04730_b200 import TcError
    ran = 0
    for name in ["2fcrelu_small", "mlp3_small", "mlp3_paper", "mlp1_ragged", "2fcrelu_paper"]:
        case, ins, seeded = case_inputs(oracle, golden, name)
        o = {"block_shape": [1, 1, 1], "fusion_strategy": "max", "rng_seed": 0,
             "shared_memory_budget": 49152, "thread_shape": [threads, 1, 1], "tile_sizes": [rows, cn, 1],
             "unroll_copy_shared": False, "unroll_factor": 1, "use_private": False, "use_shared": True}
        try:
            got, _ = run_on_gpu(engine, case["def"], ins, seeded, options=o)
        except TcError as e:
            assert e.kind == "MappingInvalid", str(e)
            continue
        ran += 1
        for k, rec in case["outputs"].items():
            assert_exact(oracle, name, k, got[k], rec["fnv"])
    assert ran >= 3


@pytest.mark.parametrize("rows,cn,threads", [(8, 8, 128), (4, 8, 64), (8, 4, 256), (3, 3, 96), (16, 8, 128),
                                             (1, 1, 64), (8, 16, 64), (8, 8, 64), (2, 2, 32)])
def test_fc_tma_variants(engine, oracle, golden, rows, cn, threads):
    """The cluster kernel with layer 0 streamed in by TMA tensor copies in
    256-step chunks (fc_tma.cu, tile_sizes[2] == 6): ragged rows (zero-filled
    boxes), column slices past the layer width, the K % 32 tail box, several
    passes per CTA when threads < rows x columns, non-portable clusters.
    Single-layer chains (MLP1) are rejected with MappingInvalid."""
    from paper_1802_04730_b200 import TcError
    ran = 0
    for name in ["2fcrelu_small", "mlp3_small", "mlp3_paper", "mlp1_ragged", "mlp1_small", "2fcrelu_paper",
                 "mlp1_paper"]:
        case, ins, seeded = case_inputs(oracle, golden, name)
        o = {"block_shape": [1, 1, 1], "fusion_strategy": "max", "rng_seed": 0,
             "shared_memory_budget": 49152, "thread_shape": [threads, 1, 1], "tile_sizes": [rows, cn, 6],
             "unroll_copy_shared": False, "unroll_factor": 1, "use_private": False, "use_shared": True}
        try:
            got, h = run_on_gpu(engine, case["def"], ins, seeded, options=o)
        except TcError as e:
            assert e.kind == "MappingInvalid", str(e)
            continue
        assert case["def"] != "MLP1"
        assert "tma-chunks" in engine.describe(h)["kernel"]
        ran += 1
        for k, rec in case["outputs"].items():
            assert_exact(oracle, f"{name}/tma{rows}x{cn}x{threads}", k, got[k], rec["fnv"])
    assert ran >= 2


@pytest.mark.parametrize("rows", [1, 2, 4])
def test_fc_regs_variants(engine, oracle, golden, rows):
    """Register-resident FC chains (fc_regs.cu, tile_sizes[2] == 2) at 1, 2 and
    4 rows per CTA (ragged last CTA), bit-exact on every golden FC case they
    take; defs with a reduction > 128 (layer 1 of MLP1/2FCRelu) are rejected
    with MappingInvalid."""
    from paper_1802_04730_b200 import TcError
    ran = 0
    for name in ["2fcrelu_small", "mlp3_small", "mlp3_paper", "mlp1_ragged", "2fcrelu_paper", "mlp1_paper"]:
        case, ins, seeded = case_inputs(oracle, golden, name)
        o = {"block_shape": [1, 1, 1], "fusion_strategy": "max", "rng_seed": 0,
             "shared_memory_budget": 49152, "thread_shape": [64, 1, 1], "tile_sizes": [rows, 1, 2],
             "unroll_copy_shared": False, "unroll_factor": 1, "use_private": False, "use_shared": True}
        try:
            got, h = run_on_gpu(engine, case["def"], ins, seeded, options=o)
        except TcError as e:
            assert e.kind == "MappingInvalid", str(e)
            assert case["def"] != "MLP3"
            continue
        assert "registers" in engine.describe(h)["kernel"]
        ran += 1
        for k, rec in case["outputs"].items():
            assert_exact(oracle, name, k, got[k], rec["fnv"])
    assert ran >= 4


@pytest.mark.parametrize("dchunk,threads", [(1, 64), (3, 128), (8, 256), (16, 512)])
def test_kru_chunks(engine, oracle, golden, dchunk, threads):
    case, ins, seeded = case_inputs(oracle, golden, "kru_paper_m8")
    o = {"block_shape": [1, 1, 1], "fusion_strategy": "max", "rng_seed": 0, "shared_memory_budget": 49152,
         "thread_shape": [threads, 1, 1], "tile_sizes": [dchunk, 1, 1], "unroll_copy_shared": False,
         "unroll_factor": 1, "use_private": False, "use_shared": True}
    got, _ = run_on_gpu(engine, "3KRU", ins, seeded, options=o)
    for k, rec in case["outputs"].items():
        assert_exact(oracle, "kru", k, got[k], rec["fnv"])


@pytest.mark.parametrize("th,rf,rw", [(1, 4, 7), (4, 4, 7), (2, 8, 7), (4, 4, 4), (4, 4, 8), (2, 8, 4),
                                      (8, 2, 7), (1, 1, 1)])
def test_gconv_variants(engine, oracle, golden, th, rf, rw):
    from paper_1802_04730_b200 import TcError
    ran = 0
    for name in ["gconv_small", "gconv_paper_n1g2"]:
        case, ins, seeded = case_inputs(oracle, golden, name)
        o = {"block_shape": [1, 1, 1], "fusion_strategy": "max", "rng_seed": 0, "shared_memory_budget": 49152,
             "thread_shape": [1, 1, 1], "tile_sizes": [th, rf, rw], "unroll_copy_shared": False,
             "unroll_factor": 1, "use_private": False, "use_shared": True}
        try:
            got, _ = run_on_gpu(engine, "gconv", ins, seeded, options=o)
        except TcError as e:  # e.g. a CTA over 512 threads: rejected, never run
            assert e.kind == "MappingInvalid", str(e)
            continue
        ran += 1
        assert_exact(oracle, name, "O", got["O"], case["outputs"]["O"]["fnv"])
    assert ran >= 1


def test_kru_full_paper_shape(engine, oracle):
    """3-KRU at M=256, N=16, D=32 against the restatement."""
    rng = oracle.rng(7)
    ins = {"W0": rng.f32((32, 16)), "W1": rng.f32((32, 16)), "W2": rng.f32((32, 16)),
           "X": rng.f32((256, 16, 16, 16))}
    got, _ = run_on_gpu(engine, "3KRU", ins, {})
    y, xw1, xw2 = oracle.kru3(ins["W0"], ins["W1"], ins["W2"], ins["X"])
    for k, ref in (("Y", y), ("XW1", xw1), ("XW2", xw2)):
        assert max_rel(ref, got[k]) <= TOL
        np.testing.assert_array_equal(got[k], ref)


def test_gconv_full_paper_shape_sampled(engine, oracle):
    """gconv at the BASELINE shape (N=32,G=32,C=F=16,58x58,3x3): the full
    oracle takes minutes, so compare 200k random output points exactly."""
    rng = oracle.rng(11)
    ins = {"I": rng.f32((32, 32, 16, 58, 58)), "W1": rng.f32((32, 16, 16, 3, 3)), "B": rng.f32((16,))}
    got, _ = run_on_gpu(engine, "gconv", ins, {})
    O = got["O"]
    assert O.shape == (32, 32, 16, 56, 56)
    idx = np.random.default_rng(0).integers(0, O.size, 200_000)
    ref = oracle.gconv_points(ins["I"], ins["W1"], ins["B"], idx)
    np.testing.assert_array_equal(O.reshape(-1)[idx], ref)


def test_c3_accumulates_in_place(engine, oracle, golden):
    """C3 is `+=` (in/out): running twice accumulates twice."""
    case, ins, seeded = case_inputs(oracle, golden, "c3_small")
    p = [to_dev(ins["I3"]), to_dev(ins["W"])]
    c3 = to_dev(seeded["C3"])
    h = engine.compile("C3", p, [c3])
    engine.run(h, p, [c3])
    engine.run(h, p, [c3])
    once = oracle.c3(ins["I3"], ins["W"], seeded["C3"])
    twice = oracle.c3(ins["I3"], ins["W"], once)
    np.testing.assert_array_equal(c3.cpu().numpy(), twice)


@pytest.mark.parametrize("name", ["tbmm_small", "c3_small", "mlp3_small", "2lut_small", "gconv_small"])
def test_host_buffers_equal_device(engine, oracle, golden, name):
    """TCB_HOST tensors (library does H2D/D2H) give the device path's bits."""
    case, ins, seeded = case_inputs(oracle, golden, name)
    got_h, _ = run_on_gpu(engine, case["def"], ins, seeded, host=True)
    for k, rec in case["outputs"].items():
        assert_exact(oracle, name + "/host", k, got_h[k], rec["fnv"])


def _pinned(a, misalign=False):
    """A pinned host tensor holding a; misalign: a view 4 bytes into its buffer."""
    t = torch.from_numpy(np.ascontiguousarray(a))
    if not misalign:
        return t.pin_memory()
    buf = torch.empty(t.numel() + 1, dtype=t.dtype).pin_memory()
    v = buf[1:].view(t.shape)
    v.copy_(t)
    return v


@pytest.mark.parametrize("misalign", [False, True])
@pytest.mark.parametrize("name", ["tbmm_small", "mlp3_small", "2fcrelu_small", "2lut_small", "kru_small"])
def test_pinned_host_buffers(engine, oracle, golden, name, misalign):
    """Pinned host tensors move by the one-launch segment copy (aligned: int4,
    misaligned: 4-byte units); sync, async and prepared runs give the
    golden bits."""
    case, ins, seeded = case_inputs(oracle, golden, name)
    d = case["def"]
    params = [_pinned(ins[n], misalign) for n in PARAM_ORDER[d]]
    given = [seeded[r].shape if r in seeded else None for r in RETURN_ORDER[d]]
    shapes = engine.infer_output_tensor_info(d, params, given)
    outs = [_pinned(seeded[r] if r in seeded else np.zeros(s, np.float32), misalign)
            for r, s in zip(RETURN_ORDER[d], shapes)]
    h = engine.compile(d, params, outs)
    engine.run(h, params, outs)
    for r, o in zip(RETURN_ORDER[d], outs):
        assert_exact(oracle, name + "/pinned", r, o.numpy(), case["outputs"][r]["fnv"])
    if seeded:  # in-out returns accumulate: restore before rerunning
        return
    s = torch.cuda.Stream()
    pr = engine.prepare(h, params, outs)
    for o in outs:
        o.zero_()
    pr.run(stream=s.cuda_stream, sync=False)
    s.synchronize()
    engine.check(h)
    for r, o in zip(RETURN_ORDER[d], outs):
        assert_exact(oracle, name + "/pinned-async", r, o.numpy(), case["outputs"][r]["fnv"])


def test_pinned_host_large_tensor_dma(engine, oracle):
    """Host tensors above the segment-copy limit (1 MiB) take the DMA path in
    the same call as small ones."""
    rng = np.random.default_rng(7)
    X = rng.uniform(-1, 1, (500, 26, 72)).astype(np.float32)  # 3.7 MB: DMA
    Y = rng.uniform(-1, 1, (500, 26, 72)).astype(np.float32)
    Xs, Ys = X[:4], Y[:4]  # small: segment copy
    for a, b in ((X, Y), (Xs, Ys)):
        pa, pb = _pinned(a), _pinned(b)
        z = torch.zeros(a.shape[0], 26, 26).pin_memory()
        engine.run(engine.compile("tbmm", [pa, pb], [z]), [pa, pb], [z])
        np.testing.assert_array_equal(z.numpy(), oracle.tbmm(a, b))


def test_host_calls_back_to_back(engine, oracle):
    """Large host calls (DMA) on pageable and pinned buffers, and async
    prepared calls of one handle queued back to back on one stream, give the
    exact result (the handle's staging buffers are reused in stream order)."""
    rng = np.random.default_rng(11)
    X = rng.uniform(-1, 1, (500, 26, 72)).astype(np.float32)
    Y = rng.uniform(-1, 1, (500, 26, 72)).astype(np.float32)
    ref = oracle.tbmm(X, Y)
    z = np.zeros((500, 26, 26), np.float32)  # pageable numpy
    h = engine.compile("tbmm", [X, Y], [z])
    engine.run(h, [X, Y], [z])
    np.testing.assert_array_equal(z, ref)
    pa, pb, pz = _pinned(X), _pinned(Y), torch.zeros(500, 26, 26).pin_memory()
    X2 = rng.uniform(-1, 1, X.shape).astype(np.float32)
    pa2, pz2 = _pinned(X2), torch.zeros(500, 26, 26).pin_memory()
    s = torch.cuda.Stream()
    r1, r2 = engine.prepare(h, [pa, pb], [pz]), engine.prepare(h, [pa2, pb], [pz2])
    for _ in range(3):
        pz.zero_()
        pz2.zero_()
        r1.run(stream=s.cuda_stream, sync=False)
        r2.run(stream=s.cuda_stream, sync=False)
        s.synchronize()
        np.testing.assert_array_equal(pz.numpy(), ref)
        np.testing.assert_array_equal(pz2.numpy(), oracle.tbmm(X2, Y))


@pytest.mark.parametrize("name,shapes", [("tbmm", [(500, 26, 72), (500, 26, 72)]),
                                         ("2FCRelu", [(128, 1128), (128, 1128), (128,), (64, 128), (64,)])])
def test_async_host_runs_pipelined(engine, oracle, name, shapes):
    """Async host runs of one handle on alternating streams with no host wait
    in between (the bench's pipelined e2e): the handle alternates between two
    device staging sets and each set's reuse waits for its previous run, so
    five in-flight runs with five different inputs all return their own exact
    results."""
    rng = np.random.default_rng(5)
    sets = [[rng.uniform(-1, 1, sh).astype(np.float32) for sh in shapes] for _ in range(5)]
    outs_np = engine.infer_output_tensor_info(name, sets[0])
    pins = [[_pinned(x) for x in ins] for ins in sets]
    pouts = [[torch.zeros(tuple(sh)).pin_memory() for sh in outs_np] for _ in sets]
    h = engine.compile(name, pins[0], pouts[0])
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    runs = [engine.prepare(h, p, o) for p, o in zip(pins, pouts)]
    for rep in range(3):
        for o in pouts:
            for t in o:
                t.zero_()
        for i, r in enumerate(runs):
            r.run(stream=streams[i % 2].cuda_stream, sync=False)
        for st in streams:
            st.synchronize()
        for ins, o in zip(sets, pouts):
            if name == "tbmm":
                refs = [oracle.tbmm(*ins)]
            else:
                o1 = oracle.fc_relu(ins[0], ins[1], ins[2])
                refs = [o1, oracle.fc_relu(o1, ins[3], ins[4])]
            for got, ref in zip(o, refs):
                np.testing.assert_array_equal(got.numpy(), ref)


def test_lut_index_out_of_range(engine):
    from paper_1802_04730_b200 import TcError
    lut = to_dev(np.ones((5, 8), np.float32))
    idx = to_dev(np.array([[0, 1], [2, 9]], np.int32))
    out = torch.zeros((2, 8), device="cuda")
    h = engine.compile("1LUT", [lut, idx], [out])
    with pytest.raises(TcError) as ei:
        engine.run(h, [lut, idx], [out])
    assert ei.value.kind == "IndexOutOfRange"


def test_lut_paper_shape(engine, oracle):
    """1LUT at E=1e6 (1e7 at the paper shape is 2.5 GB/table), D=64, B=128, L=50."""
    rng = oracle.rng(3)
    lut = rng.f32((1_000_000, 64))
    idx = rng.i32((128, 50), 0, 1_000_000)
    got, _ = run_on_gpu(engine, "1LUT", {"LUT": lut, "I": idx}, {})
    np.testing.assert_array_equal(got["O"], oracle.lut(lut, idx))


@pytest.mark.parametrize("D,threads", [(256, 32), (640, 128), (512, 64), (64, 32), (1024, 32)])
def test_lut_wide_rows_small_blocks(engine, oracle, D, threads):
    """Block sizes smaller than D/4 float4 columns (explicit options): every
    column is still summed and stored (columns >= 4*blockDim
    were left unwritten), bit-exact against the oracle."""
    rng = oracle.rng(D + threads)
    lut = rng.f32((5000, D))
    idx = rng.i32((16, 7), 0, 5000)
    opts = {"block_shape": [1, 1, 1], "fusion_strategy": "max", "rng_seed": 0, "shared_memory_budget": 49152,
            "thread_shape": [threads, 1, 1], "tile_sizes": [1, 1, 1], "unroll_copy_shared": False,
            "unroll_factor": 1, "use_private": True, "use_shared": False}
    out = np.full((16, D), np.nan, np.float32)
    p, o = [to_dev(lut), to_dev(idx)], [to_dev(out)]
    h = engine.compile("1LUT", p, o, opts)
    assert f"threads={threads}" in engine.describe(h)["kernel"]
    engine.run(h, p, o)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(o[0].cpu().numpy(), oracle.lut(lut, idx))


def test_cuda_graph_capture(engine, oracle, golden):
    case, ins, seeded = case_inputs(oracle, golden, "tbmm_paper")
    p = [to_dev(ins["X"]), to_dev(ins["Y"])]
    z = torch.zeros((500, 26, 26), device="cuda")
    h = engine.compile("tbmm", p, [z])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        engine.run(h, p, [z])  # warm-up (lazy module load) outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    z.zero_()
    with torch.cuda.graph(g):
        engine.run(h, p, [z], check_errors=False)
    g.replay()
    torch.cuda.synchronize()
    assert fnv_hex(oracle, z.cpu().numpy()) == case["outputs"]["Z"]["fnv"]


def test_tuner_populates_cache_and_compile_replays(engine, oracle, golden, tmp_path):
    """tune() on the GPU: every evaluated candidate min-updates the cache;
    a later compile without options hits the cache."""
    import paper_1802_04730_b200 as tcb
    tcb.cache_purge()
    log = tmp_path / "session.jsonl"
    case, ins, seeded = case_inputs(oracle, golden, "tmm_paper")
    p = [to_dev(ins["A"]), to_dev(ins["B"])]
    c = torch.zeros((128, 256), device="cuda")
    best = engine.tune("tmm", p, [c], population=8, generations=2, seed=1, timing_iters=3,
                       session_log=str(log))
    assert tcb.cache_size() == 1
    lines = [json.loads(x) for x in log.read_text().splitlines()]
    assert len(lines) == 3
    costs = [x["best_cost"] for x in lines]
    assert all(a >= b for a, b in zip(costs, costs[1:]))  # elitist monotonicity
    h = engine.compile("tmm", p, [c])
    d = engine.describe(h)
    assert d["options_source"] == "cache"
    assert json.loads(json.dumps(d["options"])) == best
    engine.run(h, p, [c])
    torch.cuda.synchronize()
    assert fnv_hex(oracle, c.cpu().numpy()) == case["outputs"]["C"]["fnv"]
    path = str(tmp_path / "tc-cache.json")
    tcb.cache_save(path)
    tcb.cache_purge()
    h2 = engine.compile("tmm", p, [c])
    assert engine.describe(h2)["options_source"] == "default"
    tcb.cache_load(path)
    h3 = engine.compile("tmm", p, [c])
    assert engine.describe(h3)["options_source"] == "cache"
    tcb.cache_purge()


@pytest.mark.parametrize("devices", [[0, 0], "all"])
def test_tuner_parallel_device_workers(engine, oracle, golden, tmp_path, devices):
    """Candidates scored in parallel by one host thread per listed device
    (the reference's worker pool, genetic.cc:317-345). The test box has one
    GPU, so [0, 0] runs two workers on it (the code path; their timings
    interfere) and "all" one worker per visible device. Every candidate is
    scored exactly once, the workers split them, and the winner is bit-exact."""
    import paper_1802_04730_b200 as tcb
    tcb.cache_purge()
    log = tmp_path / "session.jsonl"
    case, ins, seeded = case_inputs(oracle, golden, "tbmm_paper")
    p = [to_dev(ins["X"]), to_dev(ins["Y"])]
    z = torch.zeros((500, 26, 26), device="cuda")
    best = engine.tune("tbmm", p, [z], population=10, generations=1, seed=4, timing_iters=2,
                       session_log=str(log), devices=devices)
    lines = [json.loads(x) for x in log.read_text().splitlines()]
    per = lines[-1]["scored_per_device_worker"]
    assert len(per) == (2 if devices == [0, 0] else torch.cuda.device_count())
    assert sum(per) == 20  # 2 generations x 10 genomes, each scored once
    if devices == [0, 0]:
        assert min(per) > 0
    h = engine.compile("tbmm", p, [z], best)
    engine.run(h, p, [z])
    torch.cuda.synchronize()
    assert fnv_hex(oracle, z.cpu().numpy()) == case["outputs"]["Z"]["fnv"]
    tcb.cache_purge()


def test_release_frees_handle(engine, oracle):
    """tcb_release: the handle's staging is freed and the id stops working
    (handles only grew)."""
    from paper_1802_04730_b200 import TcError
    rng = oracle.rng(6)
    A, B = rng.f32((64, 32)), rng.f32((48, 32))
    C = np.zeros((64, 48), np.float32)
    h = engine.compile("tmm", [A, B], [C])
    engine.run(h, [A, B], [C])  # host tensors: allocates the handle's staging
    np.testing.assert_array_equal(C, oracle.tmm(A, B))
    engine.release(h)
    with pytest.raises(TcError) as ei:
        engine.run(h, [A, B], [C])
    assert ei.value.kind == "Name"
    h2 = engine.compile("tmm", [A, B], [C])
    assert h2 != h


def test_paper_style_call(engine, oracle):
    """ee.tmm(A, B) allocates, compiles and runs."""
    rng = oracle.rng(5)
    A, B = rng.f32((33, 17)), rng.f32((45, 17))
    C = engine.tmm(to_dev(A), to_dev(B))
    np.testing.assert_array_equal(C.cpu().numpy(), oracle.tmm(A, B))

