"""MappingOptions and the compilation cache (CPU): byte compatibility with
the reference's formats (options.cc:82-165, cache.cc:365-439) and the
store's semantics (min-update, incumbent wins ties, checksum, version,
unknown fields, concurrent writers, history log)."""
import json
import os
import threading

import pytest

import paper_1802_04730_b200 as tcb
from paper_1802_04730_b200 import TcError

_G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
META = _G["meta"]


def test_baseline_options_byte_identical():
    for i, ref in enumerate(META["baselines"]):
        got = tcb.options_baseline(i)
        assert got == ref["json"]
        assert tcb.options_digest(got) == ref["digest"]


def test_options_round_trip_matches_reference():
    for text, ref in META["roundtrip"].items():
        assert tcb.options_normalize(text) == ref


@pytest.mark.parametrize("mutate,kind", [
    (lambda o: o.update(bogus=1), "CorruptStore"),
    (lambda o: o.pop("unroll_factor"), "CorruptStore"),
    (lambda o: o.update(block_shape=[1, 1]), "CorruptStore"),
    (lambda o: o.update(fusion_strategy="fastest"), "CorruptStore"),
    (lambda o: o.update(unroll_factor=3), "MappingInvalid"),
    (lambda o: o.update(thread_shape=[64, 32, 1]), "MappingInvalid"),
    (lambda o: o.update(tile_sizes=[0]), "MappingInvalid"),
    (lambda o: o.update(shared_memory_budget=0), "MappingInvalid"),
])
def test_options_validation(mutate, kind):
    o = json.loads(tcb.options_baseline(0))
    mutate(o)
    with pytest.raises(TcError) as ei:
        tcb.options_validate(json.dumps(o))
    assert ei.value.kind == kind


def test_reference_store_round_trips_byte_identical():
    """A store serialized by the reference library deserializes here and
    re-serializes to the same bytes (entry with the reference's target)."""
    tcb.cache_purge()
    tcb.cache_deserialize(META["store"])
    assert tcb.cache_size() == 1
    assert tcb.cache_serialize() == META["store"]
    tcb.cache_purge()


@pytest.mark.parametrize("corrupt", [
    lambda s: s.replace("FNV1A64 ", "FNV1A64 0"),
    lambda s: s.replace("TCCACHE 1", "TCCACHE 2"),
    lambda s: s.replace("TCCACHE", "TCCACHX"),
    lambda s: s[: len(s) // 2],
])
def test_corrupt_stores_are_rejected(corrupt):
    with pytest.raises(TcError) as ei:
        tcb.cache_deserialize(corrupt(META["store"]))
    assert ei.value.kind == "CorruptStore"


def test_unknown_entry_field_is_rejected():
    hdr, body, tail = META["store"].split("\n")[:3]
    j = json.loads(body)
    j["entries"][0]["extra"] = 1
    body = json.dumps(j, separators=(",", ":"), sort_keys=True)
    import ctypes
    text = f"TCCACHE 1 {len(body)}\n{body}\nFNV1A64 {fnv(body)}\n"
    with pytest.raises(TcError) as ei:
        tcb.cache_deserialize(text)
    assert ei.value.kind == "CorruptStore"


def fnv(s):
    h = 0xCBF29CE484222325
    for b in s.encode():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def opts(tile):
    o = json.loads(tcb.options_baseline(0))
    o["tile_sizes"] = tile
    o["thread_shape"] = [16, tile[0] // 2, 1]  # 2x2 micro-tile for 32-wide tiles
    return o


def test_min_update_and_incumbent_wins(engine, tmp_path):
    tcb.cache_purge()
    hist = tmp_path / "tc-history.log"
    tcb.cache_set_history(str(hist))
    shapes = [(64, 32), (48, 32)]
    engine.cache_inject("tmm", shapes, opts([32, 32, 32]), 100)
    engine.cache_inject("tmm", shapes, opts([16, 16, 32]), 150)  # worse: ignored
    assert engine.cache_lookup("tmm", shapes)["tile_sizes"] == [32, 32, 32]
    engine.cache_inject("tmm", shapes, opts([16, 32, 32]), 100)  # tie: incumbent wins
    assert engine.cache_lookup("tmm", shapes)["tile_sizes"] == [32, 32, 32]
    engine.cache_inject("tmm", shapes, opts([16, 32, 32]), 99)   # better: replaces
    assert engine.cache_lookup("tmm", shapes)["tile_sizes"] == [16, 32, 32]
    assert engine.cache_lookup("tmm", [(64, 32), (49, 32)]) is None  # shapes are part of the key
    lines = [json.loads(x) for x in hist.read_text().splitlines()]
    assert [x["cost"] for x in lines] == [100, 150, 100, 99]
    assert set(lines[0]) == {"key", "genome", "cost", "session"}
    tcb.cache_set_history("")
    # compile replays the cached options ("hit ⇒ no tuning")
    h = engine.compile("tmm", shapes)
    d = engine.describe(h)
    assert d["options_source"] == "cache" and d["options"]["tile_sizes"] == [16, 32, 32]
    p = str(tmp_path / "tc-cache.json")
    tcb.cache_save(p)
    tcb.cache_purge()
    assert engine.cache_lookup("tmm", shapes) is None
    tcb.cache_load(p)
    assert engine.cache_lookup("tmm", shapes)["tile_sizes"] == [16, 32, 32]
    text = open(p).read()
    assert text.startswith("TCCACHE 1 ") and "\nFNV1A64 " in text
    tcb.cache_purge()


def test_concurrent_writers_keep_the_minimum(engine):
    """8 threads update one slot (cache.h:82-90: single-writer section)."""
    tcb.cache_purge()
    shapes = [(32, 16), (32, 16)]
    costs = list(range(400, 0, -1))

    def writer(k):
        for c in costs[k::8]:
            engine.cache_inject("tmm", shapes, opts([32, 32, 32]), c)

    ts = [threading.Thread(target=writer, args=(k,)) for k in range(8)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    store = json.loads(tcb.cache_serialize().split("\n")[1])
    assert len(store["entries"]) == 1 and store["entries"][0]["cost"] == 1
    tcb.cache_purge()


def test_load_missing_file_is_io():
    with pytest.raises(TcError) as ei:
        tcb.cache_load("/nonexistent/tc-cache.json")
    assert ei.value.kind == "Io"
