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


class MultiDeviceDecoder:
    """One process driving several GPUs (north_star subsystem 5):
    a host batch splits into contiguous shards, one per device, and every
    device decodes its shard through its own plan -- its own streams, staging
    slots and pinned result buffers -- concurrently with the others. No
    process group and no NCCL: the shards never communicate, and the results
    merge in shard order, so the output equals one ``decode`` of the whole
    batch.

    ``devices``: CUDA device indices (default: all visible). A device may
    appear more than once (several plans on one GPU). Inputs are int8 host
    blocks (B, n_c); pass pinned arrays (``pinned_input``) for the copies to
    overlap fully. ``plan_factory(device)`` lets tests substitute the plan."""

    def __init__(self, bg, rows_used: int, cfg, devices=None, chunks: int = 12, plan_factory=None):
        from concurrent.futures import ThreadPoolExecutor

        from .decoder import Plan, _coerce_cfg

        self.cfg = _coerce_cfg(cfg)
        if devices is None:
            import torch
            devices = list(range(torch.cuda.device_count()))
        if not devices:
            raise ValueError("need at least one device")
        self.devices = [int(d) for d in devices]
        factory = plan_factory or (lambda d: Plan(bg, rows_used, self.cfg, device=d))
        self.plans = [factory(d) for d in self.devices]
        self.k = self.plans[0].k
        self.chunks = int(chunks)
        self._pool = ThreadPoolExecutor(max_workers=len(self.plans))
        self._out = [None] * len(self.plans)

    def close(self) -> None:
        self._pool.shutdown(wait=True)

    def pinned_input(self, batch: int, n_c: int) -> np.ndarray:
        """A pinned int8 host array (batch, n_c) to fill and pass to decode."""
        import torch
        return torch.empty((batch, n_c), dtype=torch.int8, pin_memory=True).numpy()

    def _run(self, i: int, part: np.ndarray) -> dict:
        plan = self.plans[i]
        b = part.shape[0]
        out = self._out[i]
        if out is None or out["iters"].shape[0] < b:
            out = self._out[i] = plan.host_outputs(max(b, 1), pinned=True)
        if b == 0:
            return {k: v[:0] for k, v in out.items()}
        view = {k: v[:b] for k, v in out.items()}
        plan.decode_host(part, chunks=max(1, min(self.chunks, b // 86)), out=view)
        return {k: v.copy() for k, v in view.items()}

    def decode(self, llrs) -> DecodeResult:
        """Decode (B, n_c) int8 blocks; same result as ``decode(llrs, bg, cfg)``."""
        from .decoder import EarlyStop, _empty_result, unpack_bits

        arr = np.asarray(llrs)
        if arr.ndim == 1:
            arr = arr[None, :]
        if arr.dtype != np.int8:
            raise ValueError("MultiDeviceDecoder takes int8 blocks")
        arr = np.ascontiguousarray(arr)
        n = len(self.plans)
        bounds = [shard_bounds(arr.shape[0], n, i) for i in range(n)]
        futs = [self._pool.submit(self._run, i, arr[lo:hi]) for i, (lo, hi) in enumerate(bounds)]
        outs = [f.result() for f in futs]  # re-raises a shard's error
        crc = self.cfg.early_stop is EarlyStop.CRC
        parts = [DecodeResult(bits=unpack_bits(o["bits"], self.k), iterations=o["iters"].astype(np.int64),
                              success=o["success"].astype(bool), syndrome_weight=o["synd"].astype(np.int64),
                              crc_ok=o["crc_ok"].astype(bool) if crc else None)
                 for o in outs if o["iters"].shape[0]]
        return merge_results(parts) if parts else _empty_result(self.k, self.cfg)


def resolve_devices(gpus: int, visible: int, world: int = 1, local_rank: int = 0) -> list[int]:
    """Devices one bench/serving process drives.

    Under a launcher (world > 1) each process owns its LOCAL_RANK device.
    Otherwise one process drives ``gpus`` devices itself (per-device plans
    and streams, no process group). Asking for more devices than are visible
    is an error, never a silent fallback to fewer."""
    if world > 1:
        if not 0 <= local_rank < max(visible, 1):
            raise ValueError(f"LOCAL_RANK {local_rank} has no visible device ({visible} visible)")
        return [int(local_rank)]
    gpus = max(1, int(gpus))
    if gpus > visible:
        raise ValueError(f"--gpus {gpus} requested but only {visible} CUDA devices are visible")
    return list(range(gpus))


def run_per_device(n: int, fn, setup=None) -> tuple[float, list]:
    """Run ``fn(i)`` for i < n on n host threads released together; returns
    (wall seconds of the slowest, [results in device order]). ``setup(i)``
    runs on the thread before the common start (e.g. set the CUDA device).
    A worker's exception is re-raised."""
    import threading
    import time

    res = [None] * n
    err = []
    bar = threading.Barrier(n + 1)

    def work(i):
        try:
            if setup is not None:
                setup(i)
        except BaseException as e:  # noqa: BLE001
            err.append(e)
        bar.wait()
        if err:
            return
        t0 = time.perf_counter()
        try:
            out = fn(i)
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            return
        res[i] = (time.perf_counter() - t0, out)

    th = [threading.Thread(target=work, args=(i,)) for i in range(n)]
    for t in th:
        t.start()
    bar.wait()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return max(r[0] for r in res), [r[1] for r in res]
