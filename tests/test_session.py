"""The product's deterministic input generator (tcb_session_inputs /
tcb_fill_uniform, restating tuner::makeSessionInputs genetic.cc:255-291)
reproduces the reference's session inputs bit-for-bit (CPU)."""
import json
import os

import numpy as np
import pytest

import paper_1802_04730_b200 as tcb

_G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
CASES = sorted(_G["cases"])


@pytest.mark.parametrize("name", CASES)
def test_session_inputs_match_reference(engine, oracle, name):
    case = _G["cases"][name]
    params, rets = engine.signature(case["def"])
    arrays = [np.empty(case["params"][p], np.int32 if case["kinds"][p] else np.float32) for p in params]
    outs = [tuple(case["seeded"][r]) if r in case["seeded"] else None for r in rets]
    engine._session_fill(case["def"], arrays, _G["seed"], outs)
    for p, a in zip(params, arrays):
        assert "%016x" % oracle.fnv(a) == case["inputs_fnv"][p], p


def test_fill_uniform_matches_oracle(oracle):
    a = tcb.fill_uniform(10000, 1234)
    b = oracle.rng(1234).f32((10000,))
    np.testing.assert_array_equal(a, b)
    i = tcb.fill_uniform(5000, 99, 0, 37, np.int32)
    j = oracle.rng(99).i32((5000,), 0, 37)
    np.testing.assert_array_equal(i, j)
    assert i.min() >= 0 and i.max() < 37
