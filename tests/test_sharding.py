"""Multi-rank batch sharding (CPU, gloo, world_size 2): each rank computes
its batch slice with the oracle standing in for the device kernels, the
output shards are all-gathered, and every rank ends with the full result,
bit-identical to the single-process oracle. Covers uneven splits
(TBMM B=7 over 2 ranks) and in/out batch inputs (MLP3's O1)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1802_04730_b200.shard import BATCH_DIMS, shard_range


def test_shard_range_balanced():
    for n in (1, 7, 500, 128):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    assert [shard_range(500, 8, r)[1] - shard_range(500, 8, r)[0] for r in range(8)] == [63] * 4 + [62] * 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from oracle_lib import Oracle
    from paper_1802_04730_b200.shard import sharded_run

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    rng = orc.rng(5)
    out = {}
    # TBMM, uneven batch
    X, Y = rng.f32((7, 5, 9)), rng.f32((7, 6, 9))
    Z = torch.zeros((7, 5, 6))
    sharded_run("tbmm", lambda i, o: o[0].copy_(torch.from_numpy(orc.tbmm(i[0].numpy(), i[1].numpy()))),
                [torch.from_numpy(X), torch.from_numpy(Y)], [Z])
    out["tbmm"] = (Z.numpy().copy(), orc.tbmm(X, Y))
    # MLP3: batch input is the in/out return O1; weights replicated
    O1 = rng.f32((9, 12))
    W = [rng.f32((8, 12)), rng.f32((8,)), rng.f32((4, 8)), rng.f32((4,)), rng.f32((2, 4)), rng.f32((2,))]
    outs = [torch.from_numpy(O1.copy()), torch.zeros((9, 8)), torch.zeros((9, 4)), torch.zeros((9, 2))]

    def mlp3(i, o):
        r = orc.mlp3(o[0].numpy(), *[x.numpy() for x in i[1:]])
        for t, v in zip(o[1:], r):
            t.copy_(torch.from_numpy(v))

    ins = [torch.zeros((9, 3))] + [torch.from_numpy(w) for w in W]
    sharded_run("MLP3", mlp3, ins, outs)
    ref = orc.mlp3(O1, *W)
    out["mlp3"] = ([o.numpy().copy() for o in outs[1:]], list(ref))
    results[rank] = out
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_gather_full_outputs():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for rank in range(world):
        got, ref = results[rank]["tbmm"]
        np.testing.assert_array_equal(got, ref)
        for g, r in zip(*results[rank]["mlp3"]):
            np.testing.assert_array_equal(g, r)


def test_every_form_has_a_batch_dimension():
    from paper_1802_04730_b200 import ExecutionEngine
    ee = ExecutionEngine()
    import paper_1802_04730_b200._lib as L
    forms = [line.split("(")[0].split()[-1] for line in L.lib.tcb_builtin_ops().decode().splitlines()
             if line.startswith("def ")]
    assert sorted(forms) == sorted(BATCH_DIMS)


def test_c_abi_shard_range_matches_python_split():
    """tcb_shard_range (the C ABI a C++ host shards with) gives the same
    balanced split as shard.py, on the operator's own batch dimension."""
    from paper_1802_04730_b200 import ExecutionEngine
    ee = ExecutionEngine()
    X = np.zeros((500, 26, 72), np.float32)
    h = ee.compile("tbmm", [X, X], [np.zeros((500, 26, 26), np.float32)])
    for w in (1, 2, 3, 4, 8):
        assert [ee.shard_range(h, r, w) for r in range(w)] == [shard_range(500, w, r) + (500,) for r in range(w)]
    g = ee.compile("gconv", [np.zeros((32, 32, 16, 58, 58), np.float32), np.zeros((32, 16, 16, 3, 3), np.float32),
                             np.zeros((16,), np.float32)], [np.zeros((32, 32, 16, 56, 56), np.float32)])
    assert ee.shard_range(g, 3, 4) == (24, 32, 32)
    m = ee.compile("MLP3", [np.zeros(s, np.float32) for s in [(128, 128), (64, 128), (64,), (32, 64), (32,),
                                                              (2, 32), (2,)]],
                   [np.zeros((128, 128), np.float32), np.zeros((128, 64), np.float32),
                    np.zeros((128, 32), np.float32), np.zeros((128, 2), np.float32)])
    assert ee.shard_range(m, 7, 8) == (112, 128, 128)
