"""Batch sharding through the C ABI on a real GPU: world
2 and 3 ranks, every rank a process bound to cuda:0 (the test box has one
GPU; NCCL refuses two ranks on one device, so the output slices are
all-gathered over gloo). Each rank runs tcb_run_shard — its balanced batch
slice of a handle compiled for the full shapes, in place on the full device
tensors — then gathers the slices; every rank must end with the full
outputs bit-identical to one unsharded tcb_run of the same inputs."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

# (form, parameter shapes, seeded return shapes (in/out), int parameters)
CASES = [
    ("tbmm", [(500, 26, 72), (500, 26, 72)], {}, ()),
    ("2FCRelu", [(128, 1128), (128, 1128), (128,), (64, 128), (64,)], {}, ()),
    ("MLP3", [(128, 128), (64, 128), (64,), (32, 64), (32,), (2, 32), (2,)], {0: (128, 128)}, ()),
    ("C3", [(128, 1024), (1000, 1024)], {0: (128, 1000)}, ()),
    ("tmm", [(128, 32), (256, 32)], {}, ()),
    ("3KRU", [(32, 16), (32, 16), (32, 16), (7, 16, 16, 16)], {}, ()),
    ("gconv", [(5, 2, 16, 12, 12), (2, 16, 16, 3, 3), (16,)], {}, ()),
    ("2LUT", [(1000, 64), (37, 9), (1000, 64), (37, 5)], {}, (1, 3)),
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(ee, form, shapes, seeded, ints, dev):
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    ps = [torch.randint(0, shapes[i - 1][0], s, generator=g, device=dev, dtype=torch.int32) if i in ints
          else torch.rand(s, generator=g, device=dev) * 2 - 1 for i, s in enumerate(shapes)]
    _, rets = ee.signature(form)
    oshapes = ee.infer_output_tensor_info(form, shapes, [seeded.get(i) for i in range(len(rets))])
    outs = [torch.rand(s, generator=g, device=dev) * 2 - 1 if i in seeded else torch.zeros(s, device=dev)
            for i, s in enumerate(oshapes)]
    return ps, outs


def _worker(rank, world, port, results):
    import torch.distributed as dist

    from paper_1802_04730_b200 import ExecutionEngine
    from paper_1802_04730_b200.shard import gather_shards

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    ee = ExecutionEngine()
    out = {}
    for form, shapes, seeded, ints in CASES:
        ps, full = _inputs(ee, form, shapes, seeded, ints, dev)
        _, shard = _inputs(ee, form, shapes, seeded, ints, dev)
        h = ee.compile(form, ps, full)
        ee.run(h, ps, full)                                   # one unsharded call
        lo, hi, n = ee.shard_range(h, rank, world)
        ee.run_shard(h, ps, shard, rank, world)               # this rank's slice only
        torch.cuda.synchronize()
        host = [t.cpu() for t in shard]
        gather_shards(form, host, n)                          # the other ranks' slices
        same = [bool(torch.equal(a, b.cpu())) for a, b in zip(host, full)]
        out[form] = (lo, hi, n, same, ee.describe(h)["kernel"])
    results[rank] = out
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shards_gathered_bit_identical(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), results), nprocs=world, join=True, start_method="spawn")
    for rank in range(world):
        for form, (lo, hi, n, same, kern) in results[rank].items():
            assert all(same), f"rank {rank}/{world} {form} ({kern}) slice [{lo},{hi}) of {n}: {same}"
    # the slices tile the batch
    for form, *_ in CASES:
        spans = sorted((results[r][form][0], results[r][form][1]) for r in range(world))
        assert spans[0][0] == 0 and spans[-1][1] == results[0][form][2]
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_run_shard_rejects_host_and_bad_rank():
    from paper_1802_04730_b200 import ExecutionEngine, TcError
    ee = ExecutionEngine()
    X, Y = torch.rand((8, 4, 8), device="cuda"), torch.rand((8, 4, 8), device="cuda")
    Z = torch.zeros((8, 4, 4), device="cuda")
    h = ee.compile("tbmm", [X, Y], [Z])
    with pytest.raises(TcError) as ei:
        ee.run_shard(h, [X, Y], [Z], 2, 2)
    assert ei.value.kind == "MappingInvalid"
    with pytest.raises(TcError) as ei:
        ee.run_shard(h, [X.cpu(), Y.cpu()], [Z.cpu()], 0, 2)
    assert ei.value.kind == "Io"
