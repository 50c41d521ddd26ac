"""GPU parity at the BASELINE configs' real sizes, and the error paths of the
host/mixed/flooding entry points.

* config 4: all 51 Z x {BG1, BG2} (102 groups x 16 codewords) in ONE mixed
  batch, against the oracle group by group;
* config 5: the slot-scale 7,488-codeword batch (BG1 rows_used=8, Z in
  {384, 352, 320}) against the oracle;
* errors are reported against the call that caused them (async host path),
  and the mixed-batch / flooding device paths reject int8 -128 like
  decode() does (decoder.py:287-288).
"""

import ctypes
import gc
import weakref

import numpy as np
import pytest
import torch

import paper_2009_05534_b200 as nr
from paper_2009_05534_b200.synth import noisy_llrs
from oracle import oracle

pytestmark = pytest.mark.gpu


def _same(res, ref):
    bad = np.flatnonzero((res.bits != ref["bits"]).any(axis=1))
    assert bad.size == 0, f"bits differ in codewords {bad[:10]}"
    assert np.array_equal(res.iterations, ref["iterations"])
    assert np.array_equal(res.success, ref["success"])
    assert np.array_equal(res.syndrome_weight, ref["syndrome_weight"])


@pytest.mark.parametrize("stop,grouped", [("none", True), ("syndrome", True), ("none", False), ("crc", True)])
def test_config4_full_mixed_batch_vs_oracle(cuda_ok, stop, grouped):
    """BASELINE config 4 at full size: 102 groups of 16 codewords, one mixed
    batch (MixedBatchDecoder), every group bit-exact against the oracle."""
    from paper_2009_05534_b200.mixed import Group, MixedBatchDecoder
    cfg = nr.DecodeConfig(max_iter=10, early_stop=stop)
    groups, data = [], []
    for bg_id in ("BG1", "BG2"):
        for z in nr.ALL_LIFTING_SIZES:
            bg = nr.load_basegraph(bg_id, z)
            _, llr = noisy_llrs(bg, bg.m_bg, 2.0, 16, seed=(int(bg_id[-1]), z))
            groups.append(Group(bg, bg.m_bg, 16))
            data.append(oracle.quantize_i8(llr, z))
    assert len(groups) == 102
    mixed = MixedBatchDecoder(groups, cfg, streams=32, grouped=grouped)
    if grouped:
        assert len(mixed.launches) < 40 and sorted(i for lg in mixed.launches for i in lg) == list(range(102))
    for rep in range(2):  # capture, then a replay
        results = mixed.decode(data)
        for g, res, blocks in zip(groups, results, data):
            ref = oracle.decode(blocks, g.bg, cfg)
            _same(res, ref)
            if stop == "crc":
                assert np.array_equal(res.crc_ok, ref["crc_ok"])


def test_decode_multi_rejects_mixed_variants(cuda_ok):
    """nrldpc_decode_multi takes only plans of one kernel variant and CTA size."""
    import ctypes
    from paper_2009_05534_b200 import _native
    cfg = nr.DecodeConfig(max_iter=3)
    a = nr.get_plan(nr.load_basegraph("BG1", 384), 46, cfg, coscheduled=True)
    b = nr.get_plan(nr.load_basegraph("BG2", 16), 42, cfg, coscheduled=True)
    P = ctypes.c_void_p * 2
    outs = [a.alloc_outputs(1), b.alloc_outputs(1)]
    x = [torch.zeros((1, a.n_c), dtype=torch.int8, device="cuda"), torch.zeros((1, b.n_c), dtype=torch.int8, device="cuda")]
    rc = _native.load().nrldpc_decode_multi(
        P(a.handle.value, b.handle.value), 2, P(*[t.data_ptr() for t in x]), (ctypes.c_int64 * 2)(1, 1),
        P(*[o["bits"].data_ptr() for o in outs]), P(*[o["iters"].data_ptr() for o in outs]),
        P(*[o["synd"].data_ptr() for o in outs]), P(*[o["success"].data_ptr() for o in outs]), None, None, None)
    with pytest.raises(ValueError, match="same kernel variant"):
        _native.check(rc)


def test_config5_slot_batch_vs_oracle(cuda_ok):
    """BASELINE config 5: 7,488 codewords (64 cell-slots x 117), BG1
    rows_used=8, Z in {384, 352, 320}, 10 fixed iterations."""
    cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
    per = 7488 // 3
    for z in (384, 352, 320):
        bg = nr.load_basegraph("BG1", z)
        _, llr = noisy_llrs(bg, 8, 3.0, per, seed=(5, z))
        blocks = oracle.quantize_i8(llr, z)
        plan = nr.get_plan(bg, 8, cfg)
        out = plan.alloc_outputs(per)
        plan.decode_device(torch.from_numpy(blocks).cuda(), out)
        torch.cuda.synchronize()
        ref = oracle.decode(blocks, bg, cfg)
        assert np.array_equal(nr.unpack_bits(out["bits"].cpu().numpy(), plan.k), ref["bits"]), z
        assert np.array_equal(out["iters"].cpu().numpy(), ref["iterations"])
        assert np.array_equal(out["synd"].cpu().numpy(), ref["syndrome_weight"])


def _blocks(bg, n, seed, ebn0=1.5):
    _, llr = noisy_llrs(bg, bg.m_bg, ebn0, n, seed=seed)
    return oracle.quantize_i8(llr, bg.z)


def test_async_error_stays_with_its_own_ticket(cuda_ok):
    """bad, ok, ok issued without waiting: the third call retires the bad
    call's slot on its behalf. The bad call must fail at its own wait, the
    other two must succeed with correct results."""
    bg = nr.load_basegraph("BG2", 128)
    cfg = nr.DecodeConfig(max_iter=6)
    plan = nr.Plan(bg, bg.m_bg, cfg)
    good = [_blocks(bg, 7, (i, 3)) for i in range(3)]
    refs = [oracle.decode(b, bg, cfg) for b in good]
    bad = good[0].copy()
    bad[3, 11] = -128
    ins = [torch.from_numpy(x).pin_memory().numpy() for x in (bad, good[1], good[2])]
    outs = [plan.host_outputs(7, pinned=True) for _ in range(3)]
    t = [plan.decode_host_async(ins[i], chunks=2, out=outs[i])[0] for i in range(3)]
    plan.host_wait(t[1])
    plan.host_wait(t[2])
    with pytest.raises(ValueError, match="at most 127"):
        plan.host_wait(t[0])
    plan.host_wait(t[0])  # reported once
    for i in (1, 2):
        assert np.array_equal(nr.unpack_bits(outs[i]["bits"], plan.k), refs[i]["bits"])
        assert np.array_equal(outs[i]["iters"], refs[i]["iterations"])
    # a synchronous call draining a bad call in flight succeeds; the bad call
    # still fails at its own wait
    tb, _ = plan.decode_host_async(ins[0], chunks=2, out=outs[0])
    res = plan.decode_host(good[2], chunks=2)
    assert np.array_equal(nr.unpack_bits(res["bits"], plan.k), refs[2]["bits"])
    with pytest.raises(ValueError, match="at most 127"):
        plan.host_wait(tb)


def test_mixed_batch_rejects_out_of_range_inputs(cuda_ok):
    from paper_2009_05534_b200.mixed import Group, MixedBatchDecoder
    cfg = nr.DecodeConfig(max_iter=4)
    shapes = [("BG1", 64), ("BG2", 384)]
    groups, data = [], []
    for bg_id, z in shapes:
        bg = nr.load_basegraph(bg_id, z)
        groups.append(Group(bg, bg.m_bg, 5))
        data.append(_blocks(bg, 5, (z, 1)))
    mixed = MixedBatchDecoder(groups, cfg, streams=2)
    ok = mixed.decode(data)
    bad = [d.copy() for d in data]
    bad[1][2, 7] = -128
    with pytest.raises(ValueError, match="at most 127"):
        mixed.decode(bad)
    wide = [d.astype(np.int32) for d in data]
    wide[0][0, 0] = 200
    with pytest.raises(ValueError, match="at most 127"):
        mixed.decode(wide)
    again = mixed.decode([d.astype(np.int32) for d in data])  # status reset per replay
    for a, b in zip(ok, again):
        assert np.array_equal(a.bits, b.bits) and np.array_equal(a.iterations, b.iterations)


def test_flooding_device_path_rejects_out_of_range(cuda_ok):
    bg = nr.load_basegraph("BG2", 16)
    blocks = _blocks(bg, 4, (16, 2))
    cfg = nr.DecodeConfig(max_iter=5)
    ref = nr.decode_flooding(blocks, bg, cfg)
    x = torch.from_numpy(blocks).cuda()
    got = nr.decode_flooding(x, bg, cfg)
    assert np.array_equal(got.bits, ref.bits)
    bad = x.clone()
    bad[1, 40] = -128
    with pytest.raises(ValueError, match="at most 127"):
        nr.decode_flooding(bad, bg, cfg)
    wide = x.to(torch.int32)
    wide[0, 3] = 300
    with pytest.raises(ValueError, match="at most 127"):
        nr.decode_flooding(wide, bg, cfg)


def test_plan_cache_is_bounded_and_releases_plans(cuda_ok, monkeypatch):
    from paper_2009_05534_b200 import decoder
    monkeypatch.setattr(decoder, "PLAN_CACHE_MAX", 3)
    cfg = nr.DecodeConfig(max_iter=3, beta=0.625)  # keys nothing else uses
    refs = []
    for z in (8, 10, 12, 14, 16, 18):
        bg = nr.load_basegraph("BG2", z)
        refs.append(weakref.ref(decoder.get_plan(bg, bg.m_bg, cfg)))
        assert len(decoder._PLAN_CACHE) <= 3
    gc.collect()
    assert sum(r() is None for r in refs) >= 3  # evicted plans were destroyed
    bg = nr.load_basegraph("BG2", 18)
    res = nr.decode(_blocks(bg, 2, (18, 0)), bg, cfg)  # the cache still works
    assert res.bits.shape == (2, 10 * 18)


@pytest.mark.parametrize("bg_id,z,rows", [("BG1", 384, 46), ("BG2", 64, 42), ("BG1", 20, 46)])
def test_float_signed_zeros_and_overflow_vs_oracle(cuda_ok, bg_id, z, rows):
    """f16/f32 engines on inputs full of -0/+0, huge magnitudes (the f16 clip
    at +-65504 binds after the subtract and the add) and ties: bit-exact
    against the oracle (which follows the reference's numpy float16/32 ops).
    The f16 engine loads -0 as +0 and treats lvc < 0 as the sign bit."""
    bg = nr.load_basegraph(bg_id, z)
    params = nr.code_params(bg, z, rows)
    rng = np.random.default_rng(z * 7 + rows)
    B = 12
    x = rng.normal(0.0, 4.0, size=(B, params.n_c))
    x[:, : 2 * z] = 0.0
    zero = rng.random(x.shape) < 0.2
    x[zero] = np.where(rng.random(zero.sum()) < 0.5, -0.0, 0.0)
    big = rng.random(x.shape) < 0.05
    x[big] = np.sign(rng.normal(size=big.sum())) * rng.uniform(3e4, 6.5e4, size=big.sum())
    x[:2] = np.where(x[:2] == 0, -0.0, x[:2])  # two codewords with every zero negative
    for prec, dt in (("f16", np.float16), ("f32", np.float32)):
        blocks = x.astype(dt)
        for stop in ("none", "syndrome"):
            cfg = nr.DecodeConfig(precision=prec, max_iter=6, early_stop=stop, beta=0.75)
            ref = oracle.decode(blocks, bg, cfg)
            got = nr.decode(blocks, bg, cfg)
            _same(got, ref)
            tr_ref, tr = [], []
            oracle.decode(blocks[:3], bg, cfg, tr_ref)
            nr.decode(blocks[:3], bg, cfg, tr)
            assert tr == tr_ref


@pytest.mark.parametrize("stop", ["none", "syndrome"])
def test_multi_shape_launch_tm_variants_vs_oracle(cuda_ok, stop):
    """Multi-shape launches of the TM variants (plans without the
    co-scheduling hint: BG1 Z=288..384 with register rows, BG1 Z=160..256,
    BG2 Z=256..384), several shapes per launch, against the oracle."""
    from paper_2009_05534_b200.mixed import Group, MixedBatchDecoder
    cfg = nr.DecodeConfig(max_iter=8, early_stop=stop)
    # same Z, different rows_used: same kernel variant and CTA size, so they
    # share launches
    shapes = [("BG1", 384, 46), ("BG1", 384, 12), ("BG1", 384, 30), ("BG1", 352, 46), ("BG1", 256, 46),
              ("BG1", 256, 9), ("BG2", 384, 42), ("BG2", 384, 20), ("BG2", 256, 42)]
    groups, data = [], []
    for i, (bg_id, z, rows) in enumerate(shapes):
        bg = nr.load_basegraph(bg_id, z)
        _, llr = noisy_llrs(bg, rows, 1.5, 5 + i, seed=(z, rows, 21))
        groups.append(Group(bg, rows, 5 + i))
        data.append(oracle.quantize_i8(llr, z))
    mixed = MixedBatchDecoder(groups, cfg, streams=4, coscheduled=False)
    assert any(len(lg) > 1 for lg in mixed.launches)
    for rep in range(2):
        for g, res, blocks in zip(groups, mixed.decode(data), data):
            _same(res, oracle.decode(blocks, g.bg, cfg))


@pytest.mark.parametrize("bg_id,z,rows,batch", [("BG1", 384, 46, 37), ("BG1", 256, 46, 20), ("BG2", 384, 42, 21),
                                                ("BG1", 320, 12, 9), ("BG2", 320, 42, 8)])
@pytest.mark.parametrize("stop", ["none", "syndrome", "crc"])
def test_bit_sliced_final_check_vs_oracle(cuda_ok, bg_id, z, rows, batch, stop):
    """The TM layout's final check packs the hard decisions into words and
    computes 32 checks per funnel-shifted word (pack_hard_tm /
    packed_parity_tm): at low Eb/N0 most codewords end with a nonzero
    syndrome, so the final weights, success flags and bits are compared
    against the oracle, on full and partial graphs and odd batches (the last
    pair has one live lane)."""
    bg = nr.load_basegraph(bg_id, z)
    _, llr = noisy_llrs(bg, rows, -1.0, batch, seed=(z, rows, batch))
    blocks = oracle.quantize_i8(llr, z)
    blocks[0] = 0  # an all-erasure codeword: zero syndrome, zero margin, not a success
    cfg = nr.DecodeConfig(max_iter=4, early_stop=stop)
    from paper_2009_05534_b200 import _native
    from paper_2009_05534_b200.decoder import get_plan
    k, t, sm = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
    _native.check(_native.load().nrldpc_plan_kernel(get_plan(bg, rows, cfg).handle, ctypes.byref(k),
                                                    ctypes.byref(t), ctypes.byref(sm)))
    assert k.value in (1, 2, 3), f"expected a TM-layout kernel, got variant {k.value}"
    ref = oracle.decode(blocks, bg, cfg)
    res = nr.decode(blocks, bg, cfg)
    _same(res, ref)
    assert (ref["syndrome_weight"] > 0).sum() >= batch // 2
    assert not res.success[0] and res.syndrome_weight[0] == 0


def test_random_parity_sweep_short():
    """tools/parity_sweep.py for 20 s with a fixed seed: random graphs, all
    51 Z, partial graphs, odd batches, every precision and stop mode, each
    case bit-exact against the oracle."""
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(root / "tools" / "parity_sweep.py"), "20", "7"], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " 0 mismatches" in r.stdout


@pytest.mark.parametrize("pinned", [False, True])
def test_decode_numpy_multi_chunk_bytes_vs_oracle(cuda_ok, pinned):
    """decode(numpy) with enough codewords for a multi-chunk host pipeline
    (nrldpc_decode_host_bytes: each chunk's words unpacked into the (B, K)
    bytes while later chunks decode), from a pageable and a pinned array,
    bit-exact against the oracle; an odd batch leaves a short last chunk."""
    bg = nr.load_basegraph("BG2", 64)
    blocks = _blocks(bg, 1001, seed=11, ebn0=1.0)
    if pinned:
        from paper_2009_05534_b200.hostmem import pinned_empty
        pin = pinned_empty(blocks.shape, torch.int8, 0).numpy()
        pin[:] = blocks
        blocks = pin
    for stop in ("none", "syndrome"):
        cfg = nr.DecodeConfig(max_iter=6, early_stop=stop)
        res = nr.decode(blocks, bg, cfg)
        assert res.bits.dtype == np.uint8 and res.bits.shape == (1001, bg.k_b * 64)
        _same(res, oracle.decode(np.asarray(blocks), bg, cfg))
