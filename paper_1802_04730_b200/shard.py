"""Batch sharding of the paper operators across ranks (one process per GPU),
SURVEY.md §8(e): every operator has an independent outer (batch/group)
dimension and no cross-shard reduction, so a rank computes its contiguous
slice of the batch with the weights replicated, writing straight into its
slice of the full output; the only collective is the final all-gather of
the output shards (torch.distributed: NCCL over NVLink on B200, gloo in
the CPU tests). Uneven splits (TBMM B=500 over 8 ranks: 63,63,63,63,62,...)
gather padded shards and trim.
"""
from __future__ import annotations

# form -> ({param index: batch dim}, {return index: batch dim}); parameters
# not listed are replicated (weights). MLP3's batch input is its in/out
# return O1.
BATCH_DIMS = {
    "tmm": ({0: 0}, {0: 0}),
    "tbmm": ({0: 0, 1: 0}, {0: 0}),
    "C3": ({0: 0}, {0: 0}),
    "MLP1": ({0: 0}, {0: 0}),
    "2FCRelu": ({0: 0}, {0: 0, 1: 0}),
    "MLP3": ({}, {0: 0, 1: 0, 2: 0, 3: 0}),
    "3KRU": ({3: 0}, {0: 0, 1: 0, 2: 0}),
    "gconv": ({0: 0}, {0: 0}),
    "2LUT": ({1: 0, 3: 0}, {0: 0, 1: 0}),
    "1LUT": ({1: 0}, {0: 0}),
}


def shard_range(n: int, world: int, rank: int):
    """Balanced contiguous split: the first n % world ranks get one extra."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def batch_extent(form, inputs, outputs):
    pin, pout = BATCH_DIMS[form]
    for i in pin:
        return inputs[i].shape[0]
    for i in pout:
        return outputs[i].shape[0]
    raise ValueError(form)


def shard_views(form, inputs, outputs, lo, hi):
    """Dim-0 slices (contiguous views) of the batched tensors; replicated
    tensors pass through."""
    pin, pout = BATCH_DIMS[form]
    ins = [t[lo:hi] if i in pin else t for i, t in enumerate(inputs)]
    outs = [t[lo:hi] if i in pout else t for i, t in enumerate(outputs)]
    return ins, outs


def gather_shards(form, outputs, n, group=None):
    """All-gathers every batched return's rank slices (padded to the
    largest shard) so each rank holds the full outputs."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(n, world, rank)
    _, pout = BATCH_DIMS[form]
    mx = shard_range(n, world, 0)[1]  # the largest shard (rank 0's)
    for i in sorted(pout):
        full = outputs[i]
        pad = torch.zeros((mx,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
        pad[: hi - lo].copy_(full[lo:hi])
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        for r, part in enumerate(parts):
            a, b = shard_range(n, world, r)
            if b > a and r != rank:
                full[a:b].copy_(part[: b - a])


def engine_sharded_run(ee, handle, form, inputs, outputs, group=None, gather=True, stream=None):
    """This rank's slice through the C ABI (tcb_run_shard on the full device
    tensors, a handle compiled for the full shapes), then the all-gather."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi, n = ee.shard_range(handle, rank, world)
    ee.run_shard(handle, inputs, outputs, rank, world, stream=stream)
    if gather and world > 1:
        gather_shards(form, outputs, n, group)
    return lo, hi


def sharded_run(form, run_shard, inputs, outputs, group=None, gather=True):
    """Runs `run_shard(ins, outs)` on this rank's batch slice, then
    all-gathers every batched return so each rank holds the full outputs.
    `inputs`/`outputs` are the full tensors on the local device."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = batch_extent(form, inputs, outputs)
    lo, hi = shard_range(n, world, rank)
    ins, outs = shard_views(form, inputs, outputs, lo, hi)
    if hi > lo:
        run_shard(ins, outs)
    if not gather or world == 1:
        return lo, hi
    _, pout = BATCH_DIMS[form]
    mx = shard_range(n, world, 0)[1]  # the largest shard (rank 0's)
    for i in sorted(pout):
        full = outputs[i]
        piece = full[lo:hi]
        pad = torch.zeros((mx,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
        pad[: hi - lo].copy_(piece)
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        for r, part in enumerate(parts):
            a, b = shard_range(n, world, r)
            if b > a:
                full[a:b].copy_(part[: b - a])
    return lo, hi
