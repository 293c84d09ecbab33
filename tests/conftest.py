import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu under gpurun)")


def _ensure_built():
    from paper_1802_04730_b200 import build as b
    b.build(verbose=False)
    from oracle_lib import build_oracle
    build_oracle()


_ensure_built()


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(HERE, "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ops_tc():
    with open(os.path.join(ROOT, "paper_1802_04730_b200", "tc", "ops.tc")) as f:
        return f.read()


@pytest.fixture()
def engine():
    from paper_1802_04730_b200 import ExecutionEngine
    return ExecutionEngine()


def golden_inputs(oracle, case, seed):
    """Regenerate a golden case's inputs with the oracle's mt19937_64
    restatement (pinned to the reference's makeSessionInputs by
    test_oracle.py): parameters in sorted-name order from one stream, seeded
    returns from seed ^ 0x5eed."""
    params = case["params"]
    kinds = case["kinds"]
    shapes = {k: tuple(v) for k, v in params.items()}
    minext = min(e for s in shapes.values() for e in s)
    rng = oracle.rng(seed)
    ins = {}
    for name in sorted(params):
        if kinds[name]:
            ins[name] = rng.i32(shapes[name], 0, minext)
        else:
            ins[name] = rng.f32(shapes[name])
    rng2 = oracle.rng(seed ^ 0x5EED)
    seeded = {n: rng2.f32(tuple(s)) for n, s in case["seeded"].items()}
    return ins, seeded


def fnv_hex(oracle, a):
    return "%016x" % oracle.fnv(np.ascontiguousarray(a))


def max_rel(ref, got):
    """maxRelError (tensor_data.cc:221-234): max |got-ref| / max(|ref|, 1)."""
    ref = np.asarray(ref, np.float64)
    got = np.asarray(got, np.float64)
    if ref.shape != got.shape:
        return float("inf")
    if ref.size == 0:
        return 0.0
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)))
