"""Generate tests/golden/golden.json (+ small .npz vectors) by running the
REFERENCE itself (oracle/_ref/libtcref.so, compiled from /root/reference by
oracle/Makefile) on the reference's own deterministic session inputs
(tuner::makeSessionInputs, genetic.cc:255-291).

Run in this container (it needs /root/reference to build oracle/_ref):
    make -C oracle ref && python tests/golden/make_golden.py

For every case the file records the input shapes, the seed, FNV-1a64
hashes of every input the reference generated (pins our mt19937_64
restatement) and of every output the reference interpreter produced
(pins the C restatement and, on the GPU, the CUDA kernels). Small cases
also store the full output vectors in <case>.npz.

Seeded returns (C3's incoming C3, MLP3's pass-through O1) are not part of
makeSessionInputs; they are filled from a second mt19937_64 stream seeded
with seed ^ 0x5eed (U[-1,1)) — see seed_returns().
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Oracle, RefLib  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(HERE))
OPS_TC = os.path.join(ROOT, "paper_1802_04730_b200", "tc", "ops.tc")

# name, def, param shapes (declaration order), seeded returns, outputs, store_full
CASES = [
    ("tmm_small", "tmm", {"A": (64, 40), "B": (48, 40)}, {}, ["C"], True),
    ("tmm_paper", "tmm", {"A": (128, 32), "B": (256, 32)}, {}, ["C"], True),
    ("tbmm_small", "tbmm", {"X": (7, 5, 9), "Y": (7, 6, 9)}, {}, ["Z"], True),
    ("tbmm_paper", "tbmm", {"X": (500, 26, 72), "Y": (500, 26, 72)}, {}, ["Z"], False),
    ("c3_small", "C3", {"I3": (6, 37), "W": (11, 37)}, {"C3": (6, 11)}, ["C3"], True),
    ("c3_small_zero", "C3", {"I3": (6, 37), "W": (11, 37)}, {}, ["C3"], True),
    ("c3_paper", "C3", {"I3": (128, 1024), "W": (1000, 1024)}, {"C3": (128, 1000)}, ["C3"], False),
    ("mlp1_small", "MLP1", {"I": (8, 40), "W1": (24, 40), "B1": (24,)}, {}, ["O1"], True),
    ("mlp1_ragged", "MLP1", {"I": (5, 30), "W1": (7, 20), "B1": (7,)}, {}, ["O1"], True),
    ("mlp1_paper", "MLP1", {"I": (128, 1128), "W1": (128, 1128), "B1": (128,)}, {}, ["O1"], False),
    ("2fcrelu_small", "2FCRelu",
     {"I": (8, 40), "W1": (24, 40), "B1": (24,), "W2": (12, 24), "B2": (12,)}, {},
     ["O1", "O2"], True),
    ("2fcrelu_paper", "2FCRelu",
     {"I": (128, 1128), "W1": (128, 1128), "B1": (128,), "W2": (64, 128), "B2": (64,)}, {},
     ["O1", "O2"], False),
    ("mlp3_small", "MLP3",
     {"I": (8, 3), "W2": (12, 20), "B2": (12,), "W3": (6, 12), "B3": (6,), "W4": (2, 6),
      "B4": (2,)}, {"O1": (8, 20)}, ["O1", "O2", "O3", "O4"], True),
    ("mlp3_paper", "MLP3",
     {"I": (128, 128), "W2": (64, 128), "B2": (64,), "W3": (32, 64), "B3": (32,),
      "W4": (2, 32), "B4": (2,)}, {"O1": (128, 128)}, ["O1", "O2", "O3", "O4"], True),
    ("kru_small", "3KRU", {"W0": (7, 3), "W1": (2, 5), "W2": (4, 6), "X": (4, 3, 5, 6)}, {},
     ["Y", "XW1", "XW2"], True),
    ("kru_paper_m8", "3KRU",
     {"W0": (32, 16), "W1": (32, 16), "W2": (32, 16), "X": (8, 16, 16, 16)}, {},
     ["Y", "XW1", "XW2"], False),
    ("gconv_small", "gconv", {"I": (2, 3, 4, 9, 10), "W1": (3, 5, 4, 3, 3), "B": (5,)}, {},
     ["O"], True),
    ("gconv_paper_n1g2", "gconv",
     {"I": (1, 2, 16, 58, 58), "W1": (2, 16, 16, 3, 3), "B": (16,)}, {}, ["O"], False),
    ("2lut_small", "2LUT", {"LUT1": (50, 8), "I1": (6, 5), "LUT2": (40, 8), "I2": (6, 7)}, {},
     ["O1", "O2"], True),
    ("1lut_small", "1LUT", {"LUT": (70, 16), "I": (9, 12)}, {}, ["O"], True),
]

SEED = 42


def seed_returns(oracle, seed, returns):
    rng = oracle.rng(seed ^ 0x5EED)
    return {n: rng.f32(s) for n, s in returns.items()}


def main(only=None):
    src = open(OPS_TC).read()
    ref = RefLib()
    orc = Oracle()
    out = {"generator": "tests/golden/make_golden.py", "seed": SEED, "cases": {}}
    path = os.path.join(HERE, "golden.json")
    if os.path.exists(path):
        out = json.load(open(path))
    for name, entry, params, seeded, outputs, full in CASES:
        if only and name not in only:
            continue
        t0 = time.time()
        kinds = {p: (1 if p.startswith("I") and entry.endswith("LUT") and p[1:].isdigit() or
                     (entry == "1LUT" and p == "I") else 0) for p in params}
        ins = ref.session(src, entry, {**params, **seeded}, SEED, list(params), kinds)
        ins.update(seed_returns(orc, SEED, seeded))
        res = ref.run(src, entry, ins, outputs)
        rec = {
            "def": entry,
            "params": {k: list(v) for k, v in params.items()},
            "seeded": {k: list(v) for k, v in seeded.items()},
            "kinds": kinds,
            "inputs_fnv": {k: "%016x" % orc.fnv(v) for k, v in ins.items()},
            "outputs": {k: {"shape": list(v.shape), "fnv": "%016x" % orc.fnv(v),
                            "head": [float(x) for x in v.reshape(-1)[:8]]}
                        for k, v in res.items()},
            "ref_seconds": round(time.time() - t0, 3),
        }
        out["cases"][name] = rec
        if full:
            np.savez_compressed(os.path.join(HERE, name + ".npz"), **res)
        print(f"{name}: {rec['ref_seconds']} s", flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)


def main_meta():
    """Reference-side byte formats: canonical TC text + lookup key per case,
    baseline MappingOptions JSON + digest, option round trips, and one
    serialized cache store (cache.cc:365-378)."""
    src = open(OPS_TC).read()
    ref = RefLib()
    path = os.path.join(HERE, "golden.json")
    out = json.load(open(path))
    meta = {"canonical": {}, "baselines": [], "roundtrip": {}, "store": None}
    for name, entry, params, seeded, outputs, full in CASES:
        canon, key = ref.key(src, entry, {**params, **seeded})
        meta["canonical"][name] = {"canonical": canon, "lookup_key": key}
    for j, d in ref.baseline_options():
        meta["baselines"].append({"json": j, "digest": d})
    probe = ('{"block_shape":[2,1,1],"fusion_strategy":"min","rng_seed":7,'
             '"shared_memory_budget":1024,"thread_shape":[32,4,1],"tile_sizes":[8,16],'
             '"unroll_copy_shared":false,"unroll_factor":8,"use_private":true,"use_shared":false}')
    meta["roundtrip"][probe] = ref.options_roundtrip(probe)
    meta["store"] = ref.cache_serialize_one(src, "tbmm", {"X": (500, 26, 72), "Y": (500, 26, 72)},
                                            meta["baselines"][0]["json"], 12345, 1700000000)
    out["meta"] = meta
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("meta written")


if __name__ == "__main__":
    if sys.argv[1:] == ["meta"]:
        main_meta()
    else:
        main(set(sys.argv[1:]) or None)
