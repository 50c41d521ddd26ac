"""Multi-rank sharding plumbing on CPU (gloo, world_size 2): the sharded
decode merged in rank order equals the single-process decode. The decode
function here is the CPU oracle, so the test exercises only the host-side
split / gather path that bench.py and decode_sharded use on GPUs."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2009_05534_b200 as nr
from paper_2009_05534_b200.shard import (assign_groups, decode_mixed_sharded, decode_sharded, group_cost,
                                         merge_results, shard_bounds)
from paper_2009_05534_b200.synth import noisy_llrs
from oracle import oracle


def _oracle_decode(llrs, bg, cfg):
    r = oracle.decode(llrs, bg, cfg, threads=1)
    return nr.DecodeResult(bits=r["bits"], iterations=r["iterations"], success=r["success"],
                           syndrome_weight=r["syndrome_weight"], crc_ok=r["crc_ok"])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, blocks, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bg = nr.load_basegraph("BG2", 16)
    res = decode_sharded(blocks, bg, nr.DecodeConfig(max_iter=8), decode_fn=_oracle_decode)
    if rank == 0:
        np.savez(out_path, bits=res.bits, iterations=res.iterations, success=res.success,
                 synd=res.syndrome_weight)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds_cover_batch_in_order():
    for batch in (0, 1, 7, 1024, 1025):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(batch, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_gloo_two_ranks_match_single_process(tmp_path):
    bg = nr.load_basegraph("BG2", 16)
    _, llr = noisy_llrs(bg, 42, 1.5, 13, seed=99)
    blocks = oracle.quantize_i8(llr, 16)
    out = tmp_path / "merged.npz"
    mp.spawn(_worker, args=(2, _free_port(), blocks, str(out)), nprocs=2, join=True)
    got = np.load(out)
    ref = _oracle_decode(blocks, bg, nr.DecodeConfig(max_iter=8))
    assert np.array_equal(got["bits"], ref.bits)
    assert np.array_equal(got["iterations"], ref.iterations)
    assert np.array_equal(got["success"], ref.success)
    assert np.array_equal(got["synd"], ref.syndrome_weight)


def test_merge_results_keeps_order():
    a = nr.DecodeResult(np.zeros((2, 3), np.uint8), np.array([1, 2]), np.array([True, False]),
                        np.array([0, 5]))
    b = nr.DecodeResult(np.ones((1, 3), np.uint8), np.array([3]), np.array([True]), np.array([0]))
    m = merge_results([a, b])
    assert m.iterations.tolist() == [1, 2, 3] and m.bits.shape == (3, 3) and m.crc_ok is None


def test_assign_groups_balances_longest_first():
    costs = [9.0, 7.0, 6.0, 5.0, 4.0, 3.0, 2.0, 1.0]
    owner = assign_groups(costs, 3)
    loads = [sum(c for c, o in zip(costs, owner) if o == r) for r in range(3)]
    assert max(loads) - min(loads) <= 2.0 and sorted(set(owner)) == [0, 1, 2]
    assert assign_groups(costs, 1) == [0] * len(costs)
    assert assign_groups(costs, 3) == owner                      # deterministic


def _mixed_worker(rank, world, port, shapes, blocks, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    groups = [(nr.load_basegraph(b, z), rows) for b, z, rows in shapes]
    res = decode_mixed_sharded(groups, blocks, nr.DecodeConfig(max_iter=6), decode_fn=_oracle_decode)
    if rank == 0:
        np.savez(out_path, **{f"b{i}": r.bits for i, r in enumerate(res)},
                 **{f"i{i}": r.iterations for i, r in enumerate(res)})
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_mixed_groups_match_single_process(tmp_path):
    shapes = [("BG1", 16, 46), ("BG2", 7, 42), ("BG1", 12, 8), ("BG2", 30, 20), ("BG2", 2, 42)]
    blocks = []
    for b, z, rows in shapes:
        bg = nr.load_basegraph(b, z)
        _, llr = noisy_llrs(bg, rows, 1.5, 5, seed=(z, rows))
        blocks.append(oracle.quantize_i8(llr, z))
    costs = [group_cost(nr.load_basegraph(b, z), rows, 5, 6) for b, z, rows in shapes]
    assert len(set(assign_groups(costs, 2))) == 2                # both ranks get work
    out = tmp_path / "mixed.npz"
    mp.spawn(_mixed_worker, args=(2, _free_port(), shapes, blocks, str(out)), nprocs=2, join=True)
    got = np.load(out)
    for i, (b, z, rows) in enumerate(shapes):
        ref = oracle.decode(blocks[i], nr.load_basegraph(b, z), nr.DecodeConfig(max_iter=6), threads=1)
        assert np.array_equal(got[f"b{i}"], ref["bits"]) and np.array_equal(got[f"i{i}"], ref["iterations"])


class _OraclePlan:
    """Stands in for a device plan: decode_host fills the result buffers from the CPU oracle."""

    def __init__(self, bg, cfg):
        self.bg, self.cfg = bg, cfg
        self.k = bg.k_b * bg.z
        self.words = (self.k + 31) // 32

    def host_outputs(self, batch, pinned=False):
        return {"bits": np.zeros((batch, self.words), np.uint32), "iters": np.zeros(batch, np.int32),
                "synd": np.zeros(batch, np.int32), "success": np.zeros(batch, np.uint8),
                "crc_ok": np.zeros(batch, np.uint8)}

    def decode_host(self, llr, chunks=4, out=None):
        ref = oracle.decode(llr, self.bg, self.cfg)
        packed = np.packbits(ref["bits"], axis=1, bitorder="little")
        packed = np.pad(packed, ((0, 0), (0, 4 * self.words - packed.shape[1])))
        out["bits"][:] = packed.view("<u4")
        out["iters"][:] = ref["iterations"]
        out["synd"][:] = ref["syndrome_weight"]
        out["success"][:] = ref["success"]
        return out


@pytest.mark.parametrize("batch,devices", [(7, [0, 1, 2]), (2, [0, 1, 2]), (5, [3])])
def test_multi_device_decoder_shards_and_merges_in_order(batch, devices):
    from paper_2009_05534_b200.shard import MultiDeviceDecoder

    bg = nr.load_basegraph("BG2", 16)
    cfg = nr.DecodeConfig(max_iter=6, early_stop="syndrome")
    _, llr = noisy_llrs(bg, bg.m_bg, 1.0, batch, seed=(batch, 9))
    blocks = oracle.quantize_i8(llr, 16)
    dec = MultiDeviceDecoder(bg, bg.m_bg, cfg, devices=devices, plan_factory=lambda d: _OraclePlan(bg, cfg))
    try:
        res = dec.decode(blocks)
    finally:
        dec.close()
    ref = oracle.decode(blocks, bg, cfg)
    assert np.array_equal(res.bits, ref["bits"])
    assert np.array_equal(res.iterations, ref["iterations"])
    assert np.array_equal(res.syndrome_weight, ref["syndrome_weight"])


def test_resolve_devices_never_falls_back_silently():
    from paper_2009_05534_b200.shard import resolve_devices
    assert resolve_devices(4, 8) == [0, 1, 2, 3]
    assert resolve_devices(1, 1) == [0]
    assert resolve_devices(8, 8, world=8, local_rank=5) == [5]   # torchrun: one device per process
    with pytest.raises(ValueError, match="only 1 CUDA devices"):
        resolve_devices(2, 1)
    with pytest.raises(ValueError, match="no visible device"):
        resolve_devices(2, 1, world=2, local_rank=1)


def test_run_per_device_times_the_slowest_and_keeps_order():
    import time as _t

    from paper_2009_05534_b200.shard import run_per_device
    seen = []
    dt, out = run_per_device(4, lambda i: (_t.sleep(0.02 * (i == 2)), i * i)[1], setup=seen.append)
    assert out == [0, 1, 4, 9] and sorted(seen) == [0, 1, 2, 3]
    assert dt >= 0.02
    with pytest.raises(RuntimeError, match="boom"):
        run_per_device(3, lambda i: (_ for _ in ()).throw(RuntimeError("boom")) if i == 1 else i)


def test_four_standin_devices_match_single_decode():
    """N=4 in one process (the bench's --gpus 4 path without torchrun): four
    stand-in device plans, shards merged in order == one decode."""
    from paper_2009_05534_b200.shard import MultiDeviceDecoder, resolve_devices

    bg = nr.load_basegraph("BG1", 16)
    cfg = nr.DecodeConfig(max_iter=5, early_stop="none")
    _, llr = noisy_llrs(bg, bg.m_bg, 1.5, 13, seed=(4, 4))
    blocks = oracle.quantize_i8(llr, 16)
    devices = resolve_devices(4, 4)
    dec = MultiDeviceDecoder(bg, bg.m_bg, cfg, devices=devices, plan_factory=lambda d: _OraclePlan(bg, cfg))
    try:
        res = dec.decode(blocks)
    finally:
        dec.close()
    ref = oracle.decode(blocks, bg, cfg)
    assert np.array_equal(res.bits, ref["bits"]) and np.array_equal(res.iterations, ref["iterations"])
