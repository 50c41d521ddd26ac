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
from paper_2009_05534_b200.shard import decode_sharded, merge_results, shard_bounds
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
