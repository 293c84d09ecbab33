"""Front end (CPU): parse/print round trip, canonical text and cache lookup
keys byte-identical to the reference's (golden meta from the reference
library), shape inference, and the reference's diagnostics."""
import json
import os

import pytest

from paper_1802_04730_b200 import ExecutionEngine, TcError

_G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
CASES = sorted(_G["cases"])


def shapes_of(case, ee=None):
    from cases import PARAM_ORDER
    return [tuple(case["params"][n]) for n in PARAM_ORDER[case["def"]]]


def outs_of(ee, case):
    _, rets = ee.signature(case["def"])
    return [tuple(case["seeded"][r]) if r in case["seeded"] else None for r in rets]


@pytest.mark.parametrize("name", CASES)
def test_canonical_text_matches_reference(engine, name):
    case = _G["cases"][name]
    ref = _G["meta"]["canonical"][name]
    canon, key = engine.canonical(case["def"], shapes_of(case), outs_of(engine, case))
    assert canon == ref["canonical"]
    # lookup key = canonical \x1f shapes \x1f target; the target descriptor
    # differs by design (B200 vs the reference emulator)
    assert key.split("\x1f")[:2] == ref["lookup_key"].split("\x1f")[:2]
    assert key.split("\x1f")[2].startswith("tc-b200/1 sm_100a")


@pytest.mark.parametrize("name", CASES)
def test_shape_inference_matches_reference(engine, name):
    case = _G["cases"][name]
    shapes = engine.infer_output_tensor_info(case["def"], shapes_of(case), outs_of(engine, case))
    _, rets = engine.signature(case["def"])
    for r, s in zip(rets, shapes):
        assert list(s) == case["outputs"][r]["shape"]


@pytest.mark.parametrize("name", CASES)
def test_compile_resolves_kernel_without_gpu(engine, name):
    """compile() = specialize + recognise + decode: no device work."""
    case = _G["cases"][name]
    h = engine.compile(case["def"], shapes_of(case), outs_of(engine, case))
    d = engine.describe(h)
    assert d["form"] == case["def"]
    assert d["options_source"] in ("default", "cache")
    assert d["flops"] > 0 and d["bytes"] > 0


def test_renaming_does_not_change_the_key(engine):
    engine.define("""
      def mymm(float(P,Q) Left, float(R,Q) Right) -> (Out) {
        Out(x,y) +=! Left(x,z) * Right(y,z)
      }""")
    a = engine.canonical("mymm", [(4, 3), (5, 3)])
    b = engine.canonical("tmm", [(4, 3), (5, 3)])
    assert a == b
    h = engine.compile("mymm", [(4, 3), (5, 3)])
    assert engine.describe(h)["form"] == "tmm"


def test_round_trip_print(engine):
    src = """def f(float(N) A, int(M) I) -> (B) {
  B(i) = A(I(i)) * 2.0 + (A(i) > 0 ? 1 : -1) where i in 0:N
}
"""
    engine.define(src)
    c1, _ = engine.canonical("f", [(7,), (7,)])
    engine.define(c1.replace("def f(", "def g("))
    c2, _ = engine.canonical("g", [(7,), (7,)])
    assert c1 == c2


@pytest.mark.parametrize("src,kind", [
    ("def f(float(N) A) -> (B) { B(i) = A(i) +  }", "Parse"),
    ("def f(float(N) A) -> (B) { B(i) = A(i) & 1 }", "Parse"),
    ("def f(float(N) A) -> (B) { }", "Parse"),
    ("def f(float(N) A, float(N) A) -> (B) { B(i) = A(i) }", "Name"),
    ("def f(float(N) A) -> (B) { B(i) = Q(i) }", "Name"),
    ("def f(float(N) A) -> (B) { A(i) = B(i) }", "Name"),
    ("def f(float(N) A) -> (B) { B(i) = fmaxf(A(i)) }", "Name"),
    ("def f(float(N) A) -> (B) { B(i) = A }", "Name"),
    ("def g(float(N) A) -> (B) { B(i) = A(i) }\ndef f(float(N) A) -> (B) { B(i) = g(A(i)) }", "UnsupportedCall"),
])
def test_definition_errors(engine, src, kind):
    with pytest.raises(TcError) as ei:
        engine.define(src)
    assert ei.value.kind == kind


@pytest.mark.parametrize("src,shapes,outs,kind", [
    # j is constrained by nothing
    ("def f(float(N) A) -> (B) { B(i,j) = A(i) }", [(4,)], None, "UnderConstrained"),
    # fcrelu with I > O: bias(j) spans [0,I) but out has O columns
    ("""def fcrelu(float(B,I) in, float(O,I) weight, float(I) bias) -> (out) {
          out(i,j) = bias(j)
          out(b,o) += in(b,i) * weight(o,i)
          out(i,j) = fmaxf(out(i,j), 0) }""", [(2, 6), (3, 6), (6,)], None, "OutOfBounds"),
    # MLP3's pass-through O1 has no shape unless the caller gives one
    (None, [(2, 3), (4, 5), (4,), (3, 4), (3,), (2, 3), (2,)], None, "MissingBinding"),
    # one size symbol bound to two extents
    ("def f(float(N) A, float(N) B) -> (C) { C(i) = A(i) + B(i) }", [(3,), (4,)], None, "ShapeMismatch"),
    ("def f(float(N) A) -> (B) { B(i) = A(i) + A(i + 1) + B(i - 1) }", [(5,)], None, "LivenessInterference"),
])
def test_specialization_errors(engine, src, shapes, outs, kind):
    name = "MLP3"
    if src is not None:
        engine.define(src)
        name = src.split("def ")[-1].split("(")[0]
    with pytest.raises(TcError) as ei:
        engine.infer_output_tensor_info(name, shapes, outs)
    assert ei.value.kind == kind


def test_unregistered_definition_has_no_kernel(engine):
    engine.define("""def sgemm(float a, float b, float(N,M) A, float(M,K) B) -> (C) {
      C(i,j) = b * C(i,j)
      C(i,j) += a * A(i,k) * B(k,j) }""")
    with pytest.raises(TcError) as ei:
        engine.compile("sgemm", [None, None, (4, 3), (3, 5)], [(4, 5)])
    assert ei.value.kind == "NoKernel"


def test_mlp1_reduction_is_min_of_extents(engine):
    """mlp1.tc: m is constrained by I(b,m) and W1(n,m): its range is min(M,N)."""
    h = engine.compile("MLP1", [(5, 30), (7, 20), (7,)])
    d = engine.describe(h)
    assert d["flops"] == 2 * 5 * 7 * 20


def test_bad_options_are_mapping_invalid(engine):
    bad = json.loads(
        '{"block_shape":[1,1,1],"fusion_strategy":"max","rng_seed":0,"shared_memory_budget":49152,'
        '"thread_shape":[16,16,1],"tile_sizes":[48,32,32],"unroll_copy_shared":false,"unroll_factor":1,'
        '"use_private":false,"use_shared":true}')
    with pytest.raises(TcError) as ei:
        engine.compile("tmm", [(64, 32), (64, 32)], options=bad)
    assert ei.value.kind == "MappingInvalid"
    bad["thread_shape"] = [64, 32, 1]  # 2048 threads
    with pytest.raises(TcError) as ei:
        engine.compile("tmm", [(64, 32), (64, 32)], options=bad)
    assert ei.value.kind == "MappingInvalid"
