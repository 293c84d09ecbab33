"""TCTN1 tensor files (tensor_data.h:52-60) and the `tcb` command-line
driver. CPU tests: byte compatibility of the file format
with the reference's own writer/reader, the error cases the reference
raises (Io on malformed / truncated / empty-extent files), CLI exit codes
(0 ok / 1 user error / 2 internal) and the cache verbs. The GPU test runs
`tcb run` end to end and compares against oracle outputs written as TCTN1."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle_lib import Oracle, RefError, RefLib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TCB = os.path.join(ROOT, "paper_1802_04730_b200", "bin", "tcb")
OPS = os.path.join(ROOT, "paper_1802_04730_b200", "tc", "ops.tc")


def cli(*args, check=None):
    r = subprocess.run([TCB, *map(str, args)], capture_output=True, text=True, timeout=120)
    if check is not None:
        assert r.returncode == check, f"tcb {' '.join(map(str, args))}: rc={r.returncode}\n{r.stdout}\n{r.stderr}"
    return r


@pytest.fixture(scope="module")
def P():
    import paper_1802_04730_b200 as P
    assert os.path.exists(TCB), "tcb CLI not built (python paper_1802_04730_b200/build.py)"
    return P


@pytest.mark.parametrize("shape,dtype", [((3, 4), np.float32), ((2, 3, 5), np.int32), ((7,), np.float32),
                                         ((1, 1, 1, 1, 2), np.float32)])
def test_tctn1_matches_reference_writer(P, tmp_path, shape, dtype):
    rng = Oracle().rng(17)
    a = rng.f32(shape) if dtype == np.float32 else rng.i32(shape, -50, 50)
    ours, theirs = tmp_path / "ours.tctn", tmp_path / "ref.tctn"
    P.tensor_file_write(ours, a)
    if RefLib.available():
        RefLib().write_tensor(theirs, a)
        assert ours.read_bytes() == theirs.read_bytes()
        assert np.array_equal(RefLib().read_tensor(ours), a)
    b = P.tensor_file_read(ours)
    assert b.dtype == a.dtype and b.shape == a.shape and np.array_equal(b.view(np.uint32), a.view(np.uint32))


def test_tctn1_errors_like_reference(P, tmp_path):
    from paper_1802_04730_b200 import TcError
    good = tmp_path / "g.tctn"
    P.tensor_file_write(good, np.arange(6, dtype=np.float32).reshape(2, 3))
    raw = good.read_bytes()
    cases = {
        "magic": b"XCTN1" + raw[5:],
        "kind": raw[:5] + b"q" + raw[6:],
        "truncated": raw[:-3],
        "empty_extent": raw[:7] + (0).to_bytes(8, "little") + raw[15:],
        "rank17": raw[:6] + bytes([17]) + raw[7:],
    }
    for name, data in cases.items():
        p = tmp_path / f"{name}.tctn"
        p.write_bytes(data)
        with pytest.raises(TcError) as ei:
            P.tensor_file_read(p)
        assert ei.value.kind == "Io", name
        if RefLib.available():
            with pytest.raises(RefError):
                RefLib().read_tensor(p)
    with pytest.raises(TcError):
        P.tensor_file_read(tmp_path / "missing.tctn")


def test_cli_check_and_exit_codes(P, tmp_path):
    assert "ok" in cli("check", OPS, check=0).stdout
    assert "tmm(A,B;C)" in cli("check", OPS, "--def", "tmm", check=0).stdout
    bad = tmp_path / "bad.tc"
    bad.write_text("def broken(float(M) A -> (B) { B(i) = A(i) }\n")
    r = cli("check", bad, check=1)
    assert "Parse" in r.stderr
    live = tmp_path / "live.tc"
    live.write_text("def t(float(N,N) a) -> (a) { a(i,j) = a(j,i) }\n")
    cli("check", live, check=1)
    cli("frobnicate", OPS, check=1)
    cli("check", tmp_path / "nope.tc", check=1)
    cli("check", check=1)


def test_cli_compile_and_bindings(P):
    r = cli("compile", OPS, "--def", "tmm", "--sizes", "M=128,K=32,N=256", check=0)
    d = json.loads(r.stdout)
    assert d["form"] == "tmm" and d["options_source"] == "default" and d["math"] == "ffma"
    r = cli("compile", OPS, "--def", "tmm", "--sizes", "M=128,N=256", check=1)
    assert "MissingBinding" in r.stderr
    # MLP3's read-only O1 is bound through its synthesized size symbols
    r = cli("compile", OPS, "--def", "MLP3", "--sizes", "B=128,M=128,O=64,N=128,P=32,Q=2,O1__0=128,O1__1=128",
            check=0)
    assert json.loads(r.stdout)["form"] == "MLP3"
    # explicit tile/threads flags
    d = json.loads(cli("compile", OPS, "--def", "tmm", "--sizes", "M=128,K=32,N=256", "--tile", "32,32,32",
                       "--threads", "16,16,1", check=0).stdout)
    assert d["options"]["tile_sizes"] == [32, 32, 32] and d["options_source"] == "explicit"
    # a tensor-core compile with a shape it cannot take is a user error
    cli("compile", OPS, "--def", "tmm", "--sizes", "M=16,K=30,N=16", "--math", "tf32", check=1)


def test_cli_cache_verbs(P, tmp_path):
    cache = tmp_path / "tc-cache.json"
    opts = json.dumps({**json.loads(P.options_baseline(0)), "tile_sizes": [32, 32, 32],
                       "thread_shape": [16, 16, 1]})
    cli("cache", "inject", OPS, "--def", "tmm", "--sizes", "M=128,K=32,N=256", "--options", opts, "--cost",
        "1234", "--cache", cache, check=0)
    cli("cache", "inject", OPS, "--def", "tbmm", "--sizes", "B=500,N=26,M=72,K=26", "--options", opts, "--cost",
        "999", "--cache", cache, check=0)
    assert cache.read_text().startswith("TCCACHE 1 ")
    lines = cli("cache", "list", "--cache", cache, check=0).stdout.strip().splitlines()
    assert len(lines) == 2 and all("injected" in ln for ln in lines)
    e = json.loads(cli("cache", "inspect", "--cache", cache, "--index", "0", check=0).stdout)
    assert e["origin"] == "injected" and e["cost_ns"] in (1234, 999)
    cli("cache", "inspect", "--cache", cache, "--index", "7", check=1)
    # compile replays the cached best options: a hit, no retuning
    r = cli("compile", OPS, "--def", "tmm", "--sizes", "M=128,K=32,N=256", "--cache", cache, check=0)
    assert json.loads(r.stdout)["options_source"] == "cache" and "cache hit" in r.stderr
    cli("cache", "purge", "--cache", cache, check=0)
    assert cli("cache", "list", "--cache", cache, check=0).stdout.strip() == ""


@pytest.mark.gpu
def test_cli_run_against_oracle(P, tmp_path):
    orc = Oracle()
    rng = orc.rng(3)
    A, B = rng.f32((64, 40)), rng.f32((96, 40))
    P.tensor_file_write(tmp_path / "A.tctn", A)
    P.tensor_file_write(tmp_path / "B.tctn", B)
    P.tensor_file_write(tmp_path / "C_ref.tctn", orc.tmm(A, B))
    r = cli("run", OPS, "--def", "tmm", "--sizes", "M=64,K=40,N=96",
            "--inputs", f"A={tmp_path / 'A.tctn'},B={tmp_path / 'B.tctn'}",
            "--outputs", f"C={tmp_path / 'C.tctn'}", "--compare", f"C={tmp_path / 'C_ref.tctn'}", "--tol", "0",
            "--profile", check=0)
    assert "0 of 6144 elements differ bitwise" in r.stdout
    assert np.array_equal(P.tensor_file_read(tmp_path / "C.tctn"), orc.tmm(A, B))
    # C3 is in/out: its incoming value comes from --inputs
    I3, W, C0 = rng.f32((8, 64)), rng.f32((24, 64)), rng.f32((8, 24))
    for n, a in (("I3", I3), ("W", W), ("C3", C0)):
        P.tensor_file_write(tmp_path / f"{n}.tctn", a)
    P.tensor_file_write(tmp_path / "C3_ref.tctn", orc.c3(I3, W, C0))
    r = cli("run", OPS, "--def", "C3", "--sizes", "B=8,WX=64,WY=24",
            "--inputs", ",".join(f"{n}={tmp_path / (n + '.tctn')}" for n in ("I3", "W", "C3")),
            "--compare", f"C3={tmp_path / 'C3_ref.tctn'}", "--tol", "0", check=0)
    assert "0 of 192 elements differ bitwise" in r.stdout
    # wrong-shape input file: ShapeMismatch, user error
    r = cli("run", OPS, "--def", "tmm", "--sizes", "M=64,K=40,N=32", "--inputs", f"A={tmp_path / 'B.tctn'}",
            check=1)
    assert "ShapeMismatch" in r.stderr
