"""Batch sharding across GPUs.

Codewords are independent (decoder.py:108-111), so a batch splits into
contiguous shards with no exchange step and no collective on the data path.
This mirrors the reference's process-pool split (harness.py:163-189), which
merges per-worker results in batch order so serial and parallel runs agree.

* ``shard_bounds(batch, world, rank)``: the contiguous [lo, hi) of one rank.
* ``decode_sharded(llrs, bg, cfg, ...)``: one process per GPU under
  torch.distributed (torchrun); every rank decodes its shard on its own
  device and rank 0 gathers the results in shard order. Only the result
  gather uses the process group (gloo or NCCL), never the decode itself.
* ``merge_results`` concatenates DecodeResults in order.
* ``assign_groups(costs, world)`` / ``decode_mixed_sharded``: a mixed batch
  of (graph, Z, rows_used) groups spread over ranks by work (SURVEY §8e:
  weight Z * sum(w_r) * iterations per codeword), longest first onto the
  least-loaded rank; rank 0 gathers every group's result in group order.
"""

from __future__ import annotations

import numpy as np

from .decoder import DecodeResult


def shard_bounds(batch: int, world: int, rank: int) -> tuple[int, int]:
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    base, extra = divmod(int(batch), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def merge_results(parts: list[DecodeResult]) -> DecodeResult:
    crc = [p.crc_ok for p in parts]
    return DecodeResult(
        bits=np.concatenate([p.bits for p in parts]),
        iterations=np.concatenate([p.iterations for p in parts]),
        success=np.concatenate([p.success for p in parts]),
        syndrome_weight=np.concatenate([p.syndrome_weight for p in parts]),
        crc_ok=None if crc[0] is None else np.concatenate(crc),
    )


def decode_sharded(llrs, bg, cfg, decode_fn=None, group=None):
    """Decode ``llrs`` (the full batch, identical on every rank) split across
    the ranks of the default process group; returns the merged result on rank
    0 and None elsewhere. ``decode_fn`` defaults to the GPU decode on this
    rank's device (tests pass the CPU oracle to exercise the plumbing)."""
    import torch.distributed as dist

    if decode_fn is None:
        from .decoder import decode as decode_fn
    arr = np.asarray(llrs)
    if arr.ndim == 1:
        arr = arr[None, :]
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_bounds(arr.shape[0], world, rank)
    part = decode_fn(arr[lo:hi], bg, cfg)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(part, gathered, dst=0, group=group)
    return merge_results(gathered) if rank == 0 else None


def group_cost(bg, rows_used: int, batch: int, max_iter: int) -> float:
    """Decode work of one group: codewords x Z x edges x iterations."""
    edges = sum(len(bg.row_entries(r)[0]) for r in range(rows_used))
    return float(batch) * bg.z * edges * max_iter


def assign_groups(costs: list[float], world: int) -> list[int]:
    """Rank of each group: longest-processing-time-first list scheduling
    (ties to the lowest rank, so the assignment is deterministic)."""
    if world < 1:
        raise ValueError("need world >= 1")
    load = [0.0] * world
    owner = [0] * len(costs)
    for i in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        r = min(range(world), key=lambda k: (load[k], k))
        owner[i] = r
        load[r] += costs[i]
    return owner


def decode_mixed_sharded(groups, llrs: list, cfg, decode_fn=None, group=None):
    """``groups``: list of (bg, rows_used); ``llrs``: one (B_i, n_c_i) array per
    group, identical on every rank. Each rank decodes the groups assigned to
    it; returns the per-group results (group order) on rank 0, None elsewhere."""
    import torch.distributed as dist

    if decode_fn is None:
        from .decoder import decode as decode_fn
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    costs = [group_cost(bg, rows, len(np.atleast_2d(x)), cfg.max_iter) for (bg, rows), x in zip(groups, llrs)]
    owner = assign_groups(costs, world)
    mine = {i: decode_fn(np.atleast_2d(llrs[i]), groups[i][0], cfg) for i in range(len(groups)) if owner[i] == rank}
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(mine, gathered, dst=0, group=group)
    if rank != 0:
        return None
    merged = {}
    for part in gathered:
        merged.update(part)
    return [merged[i] for i in range(len(groups))]
