"""GPU parity: the sm_100a decoder (through the C ABI) against the reference's
golden vectors and against the pinned C oracle at full BASELINE sizes.

Bar: bit-exact bits, iterations, success, syndrome weight, crc_ok and trace,
for the int8 fixed-point path and for the f16/f32 paths (IEEE round-to-nearest
in the reference's operation order makes the float paths exact as well).
"""

import numpy as np
import pytest
import torch

import paper_2009_05534_b200 as nr
from paper_2009_05534_b200 import _native
from paper_2009_05534_b200.synth import noisy_llrs
from oracle import oracle
from tests.golden_cases import load_cases, make_cfg

pytestmark = pytest.mark.gpu

ALL_CASES = sorted(load_cases()["cases"])


def assert_same(res, ref_bits, ref_iters, ref_succ, ref_synd, ref_crc=None):
    assert res.bits.shape == ref_bits.shape
    bad = np.flatnonzero((res.bits != ref_bits).any(axis=1))
    assert bad.size == 0, f"bits differ in codewords {bad[:10]}"
    assert np.array_equal(res.iterations, ref_iters), (res.iterations, ref_iters)
    assert np.array_equal(res.success, ref_succ)
    assert np.array_equal(res.syndrome_weight, ref_synd)
    if ref_crc is not None:
        assert np.array_equal(res.crc_ok, ref_crc)


@pytest.mark.parametrize("name", ALL_CASES)
def test_golden(cuda_ok, name):
    case = load_cases()["cases"][name]
    bg = nr.load_basegraph(case.bg, case.z)
    cfg = make_cfg(case, nr.DecodeConfig)
    trace = [] if case.trace else None
    res = (nr.decode_flooding if case.flooding else nr.decode)(case.llr, bg, cfg, trace)
    crc = case.arrays["crc_ok"].astype(bool) if "crc_ok" in case.arrays else None
    assert_same(res, case.bits(), case.arrays["iterations"], case.arrays["success"].astype(bool),
                case.arrays["syndrome_weight"], crc)
    if case.trace:
        assert trace == case.trace_list()


def test_golden_quantize(cuda_ok):
    q = load_cases()["quant"]
    bg = nr.load_basegraph("BG2", 16)
    params = nr.code_params(bg, 16, 42)
    for mode in ("int8", "f16", "f32"):
        got = nr.quantize(q["x"], nr.QuantConfig(mode=mode), params)
        assert got.dtype == q[mode].dtype
        assert np.array_equal(got.view(np.uint8), q[mode].view(np.uint8)), mode


def test_quantize_device_tensor_f32_input(cuda_ok):
    bg = nr.load_basegraph("BG1", 384)
    params = nr.code_params(bg, 384, 46)
    _, llr = noisy_llrs(bg, 46, 2.0, 8, seed=1)
    x32 = llr.astype(np.float32)
    dev = nr.quantize(torch.from_numpy(x32).cuda(), nr.QuantConfig(), params)
    assert dev.is_cuda and dev.dtype == torch.int8
    # the reference widens float32 input to float64 before scaling
    assert np.array_equal(dev.cpu().numpy(), oracle.quantize_i8(x32.astype(np.float64), 384))


def _oracle_cmp(bg, rows, cfg, llr_i8, trace=False):
    tr_ref = [] if trace else None
    ref = oracle.decode(llr_i8, bg, cfg, tr_ref)
    tr = [] if trace else None
    res = nr.decode(llr_i8, bg, cfg, tr)
    assert_same(res, ref["bits"], ref["iterations"], ref["success"], ref["syndrome_weight"],
                ref["crc_ok"])
    if trace:
        assert tr == tr_ref
    return res


def test_config2_full_batch_vs_oracle(cuda_ok):
    """BASELINE config 2: BG1 Z=384, B=1024, fixed 10 iterations."""
    bg = nr.load_basegraph("BG1", 384)
    _, llr = noisy_llrs(bg, 46, 2.0, 1024, seed=2024)
    blocks = oracle.quantize_i8(llr, 384)
    cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
    res = _oracle_cmp(bg, 46, cfg, blocks)
    assert (res.iterations == 10).all()


def test_config3_early_termination_vs_oracle(cuda_ok):
    """BASELINE config 3: BG2 Z=384 at 0.5 dB, syndrome stop, max 20."""
    bg = nr.load_basegraph("BG2", 384)
    _, llr = noisy_llrs(bg, 42, 0.5, 512, seed=3)
    blocks = oracle.quantize_i8(llr, 384)
    res = _oracle_cmp(bg, 42, nr.DecodeConfig(max_iter=20), blocks)
    assert res.iterations.min() < res.iterations.max()  # variable iteration counts


@pytest.mark.parametrize("bg_id", ["BG1", "BG2"])
def test_config4_every_lifting_size_vs_oracle(cuda_ok, bg_id):
    """BASELINE config 4 groups: all 51 Z, 16 codewords each, 10 iterations."""
    for z in nr.ALL_LIFTING_SIZES:
        bg = nr.load_basegraph(bg_id, z)
        _, llr = noisy_llrs(bg, bg.m_bg, 2.0, 16, seed=(int(bg_id[-1]), z, 4))
        blocks = oracle.quantize_i8(llr, z)
        _oracle_cmp(bg, bg.m_bg, nr.DecodeConfig(max_iter=10, early_stop="none"), blocks)
        _oracle_cmp(bg, bg.m_bg, nr.DecodeConfig(max_iter=10), blocks)


@pytest.mark.parametrize("batch", [1, 2, 3, 5, 33, 149, 301])
def test_ragged_batches(cuda_ok, batch):
    """Batches that leave half-filled lane pairs / groups / CTAs."""
    for bg_id, z in (("BG2", 16), ("BG1", 7), ("BG1", 384), ("BG2", 240)):
        bg = nr.load_basegraph(bg_id, z)
        _, llr = noisy_llrs(bg, bg.m_bg, 1.5, batch, seed=(batch, z))
        blocks = oracle.quantize_i8(llr, z)
        _oracle_cmp(bg, bg.m_bg, nr.DecodeConfig(max_iter=8), blocks)


@pytest.mark.parametrize("bg_id,z,early", [("BG1", 384, "none"), ("BG2", 384, "syndrome"),
                                           ("BG1", 288, "syndrome"), ("BG2", 52, "none")])
def test_large_batch_position_invariance(cuda_ok, bg_id, z, early):
    """A batch of many waves (ragged count): every codeword's result is
    independent of where it sits in the batch and of its lane partner. A
    block of distinct codewords is tiled with a shift so each one lands in
    both lanes of a pair and in the first and last waves; the first tile is
    pinned against the oracle."""
    bg = nr.load_basegraph(bg_id, z)
    cfg = nr.DecodeConfig(max_iter=6, early_stop=early)
    _, llr = noisy_llrs(bg, bg.m_bg, 1.0, 37, seed=(z, 99))
    base = oracle.quantize_i8(llr, z)
    reps = 4111 // len(base) + 1
    tiled = np.concatenate([np.roll(base, i, axis=0) for i in range(reps)])[:4111]
    res = nr.decode(tiled, bg, cfg)
    ref = oracle.decode(base, bg, cfg)
    for i in range(reps):
        lo, hi = i * len(base), min((i + 1) * len(base), len(tiled))
        idx = (np.arange(lo, hi) - lo - i) % len(base)       # row of base at each position
        assert np.array_equal(res.bits[lo:hi], ref["bits"][idx]), i
        assert np.array_equal(res.iterations[lo:hi], ref["iterations"][idx]), i
        assert np.array_equal(res.syndrome_weight[lo:hi], ref["syndrome_weight"][idx]), i


def test_empty_batch(cuda_ok):
    bg = nr.load_basegraph("BG2", 16)
    res = nr.decode(np.zeros((0, 832), np.int8), bg, nr.DecodeConfig())
    assert res.bits.shape == (0, 160) and res.iterations.shape == (0,)


@pytest.mark.parametrize("rows", [4, 5, 6, 7, 8, 17, 23, 30, 45])
def test_partial_rows_vs_oracle(cuda_ok, rows):
    # BG1 Z=384 / 288: register-row kernels (rows 0..min(rows,6)-1 from
    # registers, the rest as units, a pair cut in half at odd rows_used)
    for bg_id, z in (("BG1", 384), ("BG1", 288), ("BG2", 44)):
        bg = nr.load_basegraph(bg_id, z)
        if rows > bg.m_bg:
            continue
        _, llr = noisy_llrs(bg, rows, 2.5, 24, seed=(rows, z))
        _oracle_cmp(bg, rows, nr.DecodeConfig(max_iter=12), oracle.quantize_i8(llr, z))


@pytest.mark.parametrize("beta", [0.75, 0.5, 1.0, 0.8, 0.3, 0.6875])
def test_beta_values_vs_oracle(cuda_ok, beta):
    bg = nr.load_basegraph("BG1", 104)
    _, llr = noisy_llrs(bg, 46, 1.75, 64, seed=int(beta * 1000))
    _oracle_cmp(bg, 46, nr.DecodeConfig(max_iter=15, beta=beta), oracle.quantize_i8(llr, 104))


@pytest.mark.parametrize("bg_id,z,rows,beta", [("BG1", 384, 46, 0.7), ("BG2", 384, 42, 0.55),
                                               ("BG1", 320, 20, 0.3)])
def test_table_only_beta_large_z_vs_oracle(cuda_ok, bg_id, z, rows, beta):
    """Betas without an exact half-arithmetic rule run the generic schedule
    with the table rule; still bit-exact at the largest lifting sizes."""
    bg = nr.load_basegraph(bg_id, z)
    _, llr = noisy_llrs(bg, rows, 2.0, 6, seed=(z, rows))
    _oracle_cmp(bg, rows, nr.DecodeConfig(max_iter=8, beta=beta), oracle.quantize_i8(llr, z))


def test_trace_and_crc_vs_oracle(cuda_ok):
    bg = nr.load_basegraph("BG1", 64)
    params = nr.code_params(bg, 64, 46)
    rng = np.random.default_rng(12)
    msgs = np.stack([nr.crc_attach(rng.integers(0, 2, params.k - 24, dtype=np.uint8), k=params.k)
                     for _ in range(40)])
    tx = nr.encode_batch(msgs, bg, 64, 46)[:, 128:]
    sigma = nr.ebn0_to_sigma(1.5, params.k / params.n_tx)
    llr = nr.demap_llr(nr.bpsk_awgn(tx, sigma, rng), sigma)
    blocks = oracle.quantize_i8(llr, 64)
    _oracle_cmp(bg, 46, nr.DecodeConfig(max_iter=12, early_stop="crc"), blocks, trace=True)
    _oracle_cmp(bg, 46, nr.DecodeConfig(max_iter=12, early_stop="crc", rho=4), blocks, trace=True)
    _oracle_cmp(bg, 46, nr.DecodeConfig(max_iter=7, early_stop="none"), blocks, trace=True)


def test_saturated_inputs_and_erasures(cuda_ok):
    """+-127 everywhere, all-zero blocks and mixed erasures."""
    bg = nr.load_basegraph("BG1", 384)
    rng = np.random.default_rng(9)
    blocks = rng.choice(np.array([-127, 127, 0], np.int8), size=(6, 26112))
    blocks[0] = 0
    blocks[1] = 127
    blocks[2] = -127
    _oracle_cmp(bg, 46, nr.DecodeConfig(max_iter=6), blocks)
    _oracle_cmp(bg, 46, nr.DecodeConfig(max_iter=6, early_stop="none"), blocks, trace=True)


def test_device_tensor_input_and_host_path_agree(cuda_ok):
    bg = nr.load_basegraph("BG1", 384)
    _, llr = noisy_llrs(bg, 46, 2.0, 70, seed=77)
    blocks = oracle.quantize_i8(llr, 384)
    cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
    a = nr.decode(blocks, bg, cfg)
    b = nr.decode(torch.from_numpy(blocks).cuda(), bg, cfg)
    assert np.array_equal(a.bits, b.bits) and np.array_equal(a.iterations, b.iterations)
    plan = nr.get_plan(bg, 46, cfg)
    h = plan.decode_host(blocks, chunks=3)
    assert np.array_equal(nr.unpack_bits(h["bits"], plan.k), a.bits)
    assert np.array_equal(h["iters"], a.iterations)
    assert np.array_equal(h["synd"], a.syndrome_weight)


def test_out_of_range_device_input_raises(cuda_ok):
    bg = nr.load_basegraph("BG2", 16)
    x = torch.zeros((2, 832), dtype=torch.int8, device="cuda")
    x[1, 17] = -128
    with pytest.raises(ValueError, match="at most 127"):
        nr.decode(x, bg, nr.DecodeConfig())


@pytest.mark.parametrize("bg_id,z,batch", [("BG2", 16, 3), ("BG1", 384, 40), ("BG1", 13, 1)])
def test_out_of_range_host_int8_raises_and_plan_stays_usable(cuda_ok, bg_id, z, batch):
    """Host int8 input goes straight to the device; a -128 anywhere (vector or
    scalar prologue) raises the reference's ValueError, and the next call on
    the same plan decodes normally."""
    bg = nr.load_basegraph(bg_id, z)
    _, llr = noisy_llrs(bg, bg.m_bg, 2.0, batch, seed=(z, 5))
    blocks = oracle.quantize_i8(llr, z)
    bad = blocks.copy()
    bad[-1, -3] = -128
    with pytest.raises(ValueError, match="at most 127"):
        nr.decode(bad, bg, nr.DecodeConfig(max_iter=4))
    _oracle_cmp(bg, bg.m_bg, nr.DecodeConfig(max_iter=4), blocks)


def test_async_host_pipeline_matches_sync_and_reports_errors(cuda_ok):
    """nrldpc_decode_host_async / nrldpc_host_wait: two calls in flight give
    the synchronous results; a bad input fails its own wait; a third call
    retires the oldest; the plan keeps working afterwards."""
    bg = nr.load_basegraph("BG1", 384)
    cfg = nr.DecodeConfig(max_iter=5, early_stop="syndrome")
    plan = nr.get_plan(bg, 46, cfg)
    blocks = []
    for seed in range(3):
        _, llr = noisy_llrs(bg, 46, 1.5, 9 + seed, seed=(seed, 77))
        blocks.append(oracle.quantize_i8(llr, 384))
    ref = [oracle.decode(b, bg, cfg) for b in blocks]
    pinned = [torch.from_numpy(b).pin_memory().numpy() for b in blocks]
    outs = [plan.host_outputs(len(b), pinned=True) for b in blocks]
    tickets = [plan.decode_host_async(pinned[i], chunks=3, out=outs[i])[0] for i in range(2)]
    plan.host_wait(tickets[0])
    t2, _ = plan.decode_host_async(pinned[2], chunks=3, out=outs[2])
    plan.host_wait(tickets[1])
    plan.host_wait(t2)
    plan.host_wait(t2)                                   # already retired: no-op
    for i in range(3):
        assert np.array_equal(nr.unpack_bits(outs[i]["bits"], plan.k), ref[i]["bits"]), i
        assert np.array_equal(outs[i]["iters"], ref[i]["iterations"]), i
    bad = pinned[0].copy()
    bad[0, 5] = -128
    t_bad, _ = plan.decode_host_async(bad, chunks=2, out=outs[0])
    with pytest.raises(ValueError, match="at most 127"):
        plan.host_wait(t_bad)
    t_ok, _ = plan.decode_host_async(pinned[1], chunks=2, out=outs[1])
    plan.host_wait(t_ok)
    assert np.array_equal(nr.unpack_bits(outs[1]["bits"], plan.k), ref[1]["bits"])


@pytest.mark.parametrize("bg_id,z,stop,ebn0", [("BG1", 384, "syndrome", 2.0), ("BG2", 384, "crc", 1.0),
                                               ("BG1", 256, "syndrome", 1.5), ("BG2", 96, "syndrome", 0.8)])
def test_lane_refill_matches_pair_kernel_and_oracle(cuda_ok, bg_id, z, stop, ebn0, monkeypatch):
    """Early-stop modes run the persistent lane-refill kernel; it must give
    the pair kernel's (and the oracle's) results codeword for codeword."""
    bg = nr.load_basegraph(bg_id, z)
    params = nr.code_params(bg, z, bg.m_bg)
    rng = np.random.default_rng(z)
    if stop == "crc":
        msgs = np.stack([nr.crc_attach(rng.integers(0, 2, params.k - 24, dtype=np.uint8), k=params.k)
                         for _ in range(301)])
        tx = nr.encode_batch(msgs, bg, z, bg.m_bg)[:, 2 * z:]
        sigma = nr.ebn0_to_sigma(ebn0, params.k / params.n_tx)
        llr = nr.demap_llr(nr.bpsk_awgn(tx, sigma, rng), sigma)
    else:
        _, llr = noisy_llrs(bg, bg.m_bg, ebn0, 301, seed=(z, 3))
    blocks = oracle.quantize_i8(llr, z)
    cfg = nr.DecodeConfig(max_iter=12, early_stop=stop)
    res = _oracle_cmp(bg, bg.m_bg, cfg, blocks)                 # refill path (default)
    monkeypatch.setenv("NRLDPC_NO_REFILL", "1")
    res2 = nr.decode(blocks, bg, cfg)                           # pair kernel
    assert np.array_equal(res.bits, res2.bits) and np.array_equal(res.iterations, res2.iterations)
    assert len(set(res.iterations.tolist())) > 1                # lanes really refilled at different times


def test_native_library_is_the_compute_path(cuda_ok):
    bg = nr.load_basegraph("BG2", 64)
    nr.decode(np.zeros((4, 3328), np.int8), bg, nr.DecodeConfig(max_iter=2))
    assert _native.launch_count() >= 1


def test_demap_quantize_matches_reference_chain(cuda_ok):
    """Fused demapper+quantizer == channel.demap_llr then channel.quantize."""
    for bg_id, z, rows in (("BG1", 384, 46), ("BG2", 13, 42)):
        bg = nr.load_basegraph(bg_id, z)
        params = nr.code_params(bg, z, rows)
        rng = np.random.default_rng(z)
        sigma = nr.ebn0_to_sigma(1.0, params.k / params.n_tx)
        y = nr.bpsk_awgn(rng.integers(0, 2, size=(5, params.n_tx)), sigma, rng)
        ref = oracle.quantize_i8(nr.demap_llr(y, sigma), z)          # channel.py:57-61, 64-83
        got = nr.demap_quantize(y, sigma, nr.QuantConfig(), params)
        assert np.array_equal(got, ref)
        dev = nr.demap_quantize(torch.from_numpy(y).cuda(), sigma, nr.QuantConfig(), params)
        assert np.array_equal(dev.cpu().numpy(), ref)


def test_crc_at_full_size_vs_oracle(cuda_ok):
    """Group-parallel CRC-24B over K=8448 hard bits (crc table path)."""
    bg = nr.load_basegraph("BG1", 384)
    params = nr.code_params(bg, 384, 46)
    rng = np.random.default_rng(21)
    msgs = np.stack([nr.crc_attach(rng.integers(0, 2, params.k - 24, dtype=np.uint8), k=params.k)
                     for _ in range(24)])
    msgs[5, 100] ^= 1  # one codeword whose payload no longer matches its CRC
    tx = nr.encode_batch(msgs, bg, 384, 46)[:, 768:]
    sigma = nr.ebn0_to_sigma(2.5, params.k / params.n_tx)
    blocks = oracle.quantize_i8(nr.demap_llr(nr.bpsk_awgn(tx, sigma, rng), sigma), 384)
    res = _oracle_cmp(bg, 46, nr.DecodeConfig(max_iter=12, early_stop="crc"), blocks)
    assert not res.crc_ok[5] and res.crc_ok.sum() >= 4  # int8 at scale 8 converges for some


@pytest.mark.parametrize("prec", ["f32", "f16"])
def test_float_paths_vs_oracle(cuda_ok, prec):
    """f32 (one codeword per thread) and f16 (two per half2) engines: exact."""
    for bg_id, z, rows, b, stop in (("BG1", 384, 46, 6, "none"), ("BG2", 52, 42, 33, "syndrome"),
                                    ("BG1", 7, 46, 17, "syndrome"), ("BG2", 384, 20, 5, "syndrome")):
        bg = nr.load_basegraph(bg_id, z)
        params = nr.code_params(bg, z, rows)
        _, llr = noisy_llrs(bg, rows, 1.75, b, seed=(z, rows, 5))
        blocks = nr.quantize(llr, nr.QuantConfig(mode=prec), params)
        cfg = nr.DecodeConfig(precision=prec, max_iter=9, early_stop=stop)
        _oracle_cmp(bg, rows, cfg, blocks, trace=True)


def test_float_crc_vs_oracle(cuda_ok):
    bg = nr.load_basegraph("BG2", 64)
    params = nr.code_params(bg, 64, 42)
    rng = np.random.default_rng(33)
    msgs = np.stack([nr.crc_attach(rng.integers(0, 2, params.k - 24, dtype=np.uint8), k=params.k)
                     for _ in range(12)])
    tx = nr.encode_batch(msgs, bg, 64, 42)[:, 128:]
    sigma = nr.ebn0_to_sigma(1.5, params.k / params.n_tx)
    llr = nr.demap_llr(nr.bpsk_awgn(tx, sigma, rng), sigma)
    for prec in ("f32", "f16"):
        blocks = nr.quantize(llr, nr.QuantConfig(mode=prec), params)
        _oracle_cmp(bg, 42, nr.DecodeConfig(precision=prec, max_iter=12, early_stop="crc"), blocks)


def test_mixed_batch_cuda_graph_matches_per_group(cuda_ok):
    """Transport-block style mixed batch (several graphs/Z/rows in one CUDA
    graph replay) == one decode per group."""
    from paper_2009_05534_b200.mixed import Group, MixedBatchDecoder
    cfg = nr.DecodeConfig(max_iter=8)
    shapes = [("BG1", 384, 46, 6), ("BG1", 352, 8, 9), ("BG2", 13, 42, 33), ("BG2", 240, 20, 4),
              ("BG1", 2, 46, 70)]
    groups, data = [], []
    for bg_id, z, rows, b in shapes:
        bg = nr.load_basegraph(bg_id, z)
        _, llr = noisy_llrs(bg, rows, 2.0, b, seed=(z, rows, 8))
        groups.append(Group(bg, rows, b))
        data.append(oracle.quantize_i8(llr, z))
    mixed = MixedBatchDecoder(groups, cfg, streams=4)
    for _ in range(2):  # second call replays the captured graph
        results = mixed.decode(data)
        for (bg_id, z, rows, b), res, blocks in zip(shapes, results, data):
            ref = oracle.decode(blocks, nr.load_basegraph(bg_id, z), cfg)
            assert_same(res, ref["bits"], ref["iterations"], ref["success"], ref["syndrome_weight"])


@pytest.mark.parametrize("bg_id,z,rows", [("BG1", 256, 46), ("BG2", 384, 42), ("BG1", 320, 10),
                                          ("BG2", 96, 7)])
def test_coscheduled_plan_variant_is_bit_exact(cuda_ok, bg_id, z, rows):
    """The co-scheduling hint only swaps the kernel variant: same results."""
    bg = nr.load_basegraph(bg_id, z)
    cfg = nr.DecodeConfig(max_iter=6, early_stop="syndrome")
    _, llr = noisy_llrs(bg, rows, 1.5, 9, seed=(z, rows, 11))
    blocks = oracle.quantize_i8(llr, z)
    ref = oracle.decode(blocks, bg, cfg)
    for co in (False, True):
        plan = nr.Plan(bg, rows, cfg, coscheduled=co)
        x = torch.from_numpy(blocks).cuda()
        out = plan.alloc_outputs(len(blocks))
        plan.decode_device(x, out)
        bits = nr.unpack_bits(out["bits"].cpu().numpy(), plan.k)
        assert np.array_equal(bits, ref["bits"]), co
        assert np.array_equal(out["iters"].cpu().numpy(), ref["iterations"]), co


@pytest.mark.parametrize("bg_id,z,rows", [("BG1", 384, 46), ("BG2", 13, 42), ("BG1", 7, 9),
                                          ("BG2", 240, 4), ("BG1", 2, 46)])
def test_gpu_encoder_matches_host_encoder(cuda_ok, bg_id, z, rows):
    from paper_2009_05534_b200 import sim
    bg = nr.load_basegraph(bg_id, z)
    plan = nr.get_plan(bg, rows, nr.DecodeConfig())
    rng = np.random.default_rng(z)
    msgs = rng.integers(0, 2, size=(19, bg.k_b * z), dtype=np.uint8)
    got = sim.encode(torch.from_numpy(msgs).cuda(), plan).cpu().numpy()
    assert np.array_equal(got, nr.encode_batch(msgs, bg, z, rows))   # codec.py:66-139


def test_gpu_channel_statistics(cuda_ok):
    """BPSK/AWGN/demap/quantize on the GPU: punctured zeros, right LLR moments."""
    from paper_2009_05534_b200 import sim
    bg = nr.load_basegraph("BG1", 384)
    plan = nr.get_plan(bg, 46, nr.DecodeConfig())
    bits = torch.randint(0, 2, (64, plan.n_c), dtype=torch.uint8, device="cuda")
    sigma = 1.3
    q = sim.channel(bits, plan, sigma, scale=1.0, seed=7).cpu().numpy().astype(np.float64)
    b = bits.cpu().numpy()
    assert not q[:, :768].any()
    x, bb = q[:, 768:], b[:, 768:]
    mean = 2.0 / sigma ** 2                       # E[L | b=0] = 2/sigma^2, Var = 4/sigma^2
    assert abs(x[bb == 0].mean() - mean) < 0.02 and abs(x[bb == 1].mean() + mean) < 0.02
    assert abs(x[bb == 0].std() - 2.0 / sigma) < 0.03
    q2 = sim.channel(bits, plan, sigma, scale=1.0, seed=7).cpu().numpy()
    assert np.array_equal(q, q2)                  # counter-based: reproducible


def test_gpu_bler_sweep_monotone(cuda_ok):
    from paper_2009_05534_b200 import sim
    bg = nr.load_basegraph("BG2", 16)
    pts = sim.bler_sweep(bg, 42, nr.DecodeConfig(max_iter=20), [float("inf"), 0.5, 2.0, 3.5],
                         target_block_errors=100, max_codewords=4000, seed=808, batch=2000)
    assert pts[0].block_errors == 0
    for prev, nxt in zip(pts[1:], pts[2:]):
        assert nxt.wilson()[0] <= prev.wilson()[1]
    assert pts[1].bler > pts[3].bler


@pytest.mark.parametrize("prec", ["int8", "f32", "f16"])
def test_flooding_vs_oracle(cuda_ok, prec):
    for bg_id, z, rows, b in (("BG1", 384, 46, 4), ("BG2", 52, 42, 20), ("BG1", 5, 12, 9)):
        bg = nr.load_basegraph(bg_id, z)
        params = nr.code_params(bg, z, rows)
        _, llr = noisy_llrs(bg, rows, 2.0, b, seed=(z, 77))
        blocks = nr.quantize(llr, nr.QuantConfig(mode=prec), params)
        cfg = nr.DecodeConfig(precision=prec, max_iter=12)
        tr_ref, tr = [], []
        ref = oracle.decode_flooding(blocks, bg, cfg, tr_ref)
        res = nr.decode_flooding(blocks, bg, cfg, tr)
        assert_same(res, ref["bits"], ref["iterations"], ref["success"], ref["syndrome_weight"])
        assert tr == tr_ref


def test_flooding_rejects_packed(cuda_ok):
    bg = nr.load_basegraph("BG2", 16)
    with pytest.raises(ValueError, match="rho < 4"):
        nr.decode_flooding(np.zeros((4, 832), np.int8), bg, nr.DecodeConfig(rho=4))


def test_acceptance_layered_needs_fewer_iterations_than_flooding(cuda_ok):
    """Reference acceptance criterion 7 (tests/test_acceptance.py:174-199):
    BG2 Z=52 at 3 dB, f32, max 60: both >= 99% success and layered mean
    iterations <= 0.65 x flooding, here on 2000 codewords decoded on the GPU."""
    bg = nr.load_basegraph("BG2", 52)
    params = nr.code_params(bg, 52, 42)
    cfg = nr.DecodeConfig(precision="f32", max_iter=60)
    lay_it, flo_it, lay_ok, flo_ok = [], [], 0, 0
    for start in range(0, 2000, 500):
        _, llr = noisy_llrs(bg, 42, 3.0, 500, seed=(700, start))
        blocks = nr.quantize(llr, nr.QuantConfig(mode="f32"), params)
        lay = nr.decode(blocks, bg, cfg)
        flo = nr.decode_flooding(blocks, bg, cfg)
        lay_it += lay.iterations.tolist()
        flo_it += flo.iterations.tolist()
        lay_ok += int(lay.success.sum())
        flo_ok += int(flo.success.sum())
    assert lay_ok >= 0.99 * 2000 and flo_ok >= 0.99 * 2000
    assert np.mean(lay_it) <= 0.65 * np.mean(flo_it)


@pytest.mark.parametrize("prec,stop", [("int8", "syndrome"), ("f16", "none"), ("f32", "syndrome")])
def test_scratch_paths_capture_and_concurrent_streams(cuda_ok, prec, stop):
    """Launches that take stream-ordered scratch from the library pool (the
    lane-refill work counter, float message workspaces) work inside a CUDA
    graph capture and concurrently on two streams."""
    bg = nr.load_basegraph("BG1", 384)
    cfg = nr.DecodeConfig(max_iter=8, early_stop=stop, precision=prec)
    params = nr.code_params(bg, 384, 46)
    _, llr = noisy_llrs(bg, 46, 2.5, 6, seed=(len(prec), len(stop), 5))
    blocks = nr.quantize(llr, nr.QuantConfig(mode=prec), params)
    ref = oracle.decode(blocks, bg, cfg)
    plan = nr.Plan(bg, 46, cfg)
    x = torch.from_numpy(np.ascontiguousarray(blocks)).cuda()

    def check(out):
        torch.cuda.synchronize()
        bits = nr.unpack_bits(out["bits"].cpu().numpy(), plan.k)
        assert np.array_equal(bits, ref["bits"])
        assert np.array_equal(out["iters"].cpu().numpy(), ref["iterations"])

    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = [plan.alloc_outputs(len(blocks)) for _ in range(2)]
    for _ in range(3):
        for s, o in zip(streams, outs):
            s.wait_stream(torch.cuda.current_stream())
            plan.decode_device(x, o, stream=s.cuda_stream)
    for o in outs:
        check(o)

    out = plan.alloc_outputs(len(blocks))
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.decode_device(x, out, stream=s.cuda_stream)  # warm-up outside capture
        torch.cuda.synchronize()
        for v in out.values():
            v.zero_()
        with torch.cuda.graph(g, stream=s):
            plan.decode_device(x, out, stream=s.cuda_stream)
    g.replay()
    check(out)
    for v in out.values():
        v.zero_()
    g.replay()
    check(out)


@pytest.mark.parametrize("bg_id,z,rows,stop,batch", [
    ("BG1", 384, 46, "none", 64), ("BG1", 288, 46, "none", 37), ("BG1", 320, 9, "none", 20),
    ("BG1", 352, 46, "syndrome", 2), ("BG1", 384, 30, "crc", 2), ("BG1", 384, 6, "none", 8),
    ("BG1", 384, 7, "none", 8), ("BG1", 256, 46, "none", 33), ("BG1", 160, 46, "syndrome", 64),
    ("BG1", 224, 46, "none", 9), ("BG2", 384, 42, "none", 40), ("BG2", 256, 42, "syndrome", 65),
    ("BG2", 320, 42, "crc", 2)])
def test_tm_layout_matches_byte_pair_layout_and_oracle(cuda_ok, bg_id, z, rows, stop, batch, monkeypatch):
    """Single-group pair shapes that hold an SM alone decode on the TM layout
    (half2 posteriors, messages in shared and tensor memory; the lane-refill
    kernel too for early stops with batch > 2); NRLDPC_NO_TM=1 selects the
    byte-pair layout. Both must give the oracle's results."""
    monkeypatch.delenv("NRLDPC_NO_TM", raising=False)  # the first plan must take the TM layout
    bg = nr.load_basegraph(bg_id, z)
    params = nr.code_params(bg, z, rows)
    if stop == "crc":
        rng = np.random.default_rng(z)
        msgs = np.stack([nr.crc_attach(rng.integers(0, 2, params.k - 24, dtype=np.uint8), k=params.k)
                         for _ in range(batch)])
        tx = nr.encode_batch(msgs, bg, z, rows)[:, 2 * z:]
        sigma = nr.ebn0_to_sigma(1.5, params.k / params.n_tx)
        llr = nr.demap_llr(nr.bpsk_awgn(tx, sigma, rng), sigma)
    else:
        _, llr = noisy_llrs(bg, rows, 1.5, batch, seed=(z, rows))
    blocks = oracle.quantize_i8(llr, z)
    cfg = nr.DecodeConfig(max_iter=8, early_stop=stop)
    ref = oracle.decode(blocks, bg, cfg)
    outs, smem = [], []
    for no_tm in (False, True):
        if no_tm:
            monkeypatch.setenv("NRLDPC_NO_TM", "1")
        plan = nr.Plan(bg, rows, cfg)
        smem.append(plan.smem_bytes)
        out = plan.alloc_outputs(batch)
        plan.decode_device(torch.from_numpy(blocks).cuda(), out)
        torch.cuda.synchronize()
        outs.append({k: v.cpu().numpy() for k, v in out.items() if v is not None})
    assert smem[0] != smem[1]                                   # two different layouts ran
    for o in outs:
        assert np.array_equal(nr.unpack_bits(o["bits"], params.k), ref["bits"])
        assert np.array_equal(o["iters"], ref["iterations"])
        assert np.array_equal(o["synd"], ref["syndrome_weight"])
        assert np.array_equal(o["success"].astype(bool), ref["success"])


@pytest.mark.parametrize("bg_id,z,stop,batch,devices", [("BG1", 384, "none", 301, [0, 0]),
                                                        ("BG2", 384, "syndrome", 257, [0, 0, 0]),
                                                        ("BG2", 52, "crc", 2, [0, 0, 0])])
def test_multi_device_decoder_matches_single_decode(cuda_ok, bg_id, z, stop, batch, devices):
    """One process, several plans (per-device streams and pinned buffers, no
    process group): shards merge to exactly the single-call result. One GPU
    here, so the plans share device 0."""
    from paper_2009_05534_b200.shard import MultiDeviceDecoder

    bg = nr.load_basegraph(bg_id, z)
    params = nr.code_params(bg, z, bg.m_bg)
    if stop == "crc":
        rng = np.random.default_rng(z)
        msgs = np.stack([nr.crc_attach(rng.integers(0, 2, params.k - 24, dtype=np.uint8), k=params.k)
                         for _ in range(batch)])
        tx = nr.encode_batch(msgs, bg, z, bg.m_bg)[:, 2 * z:]
        sigma = nr.ebn0_to_sigma(2.0, params.k / params.n_tx)
        llr = nr.demap_llr(nr.bpsk_awgn(tx, sigma, rng), sigma)
    else:
        _, llr = noisy_llrs(bg, bg.m_bg, 1.0, batch, seed=(z, 11))
    blocks = oracle.quantize_i8(llr, z)
    cfg = nr.DecodeConfig(max_iter=10, early_stop=stop)
    dec = MultiDeviceDecoder(bg, bg.m_bg, cfg, devices=devices)
    try:
        pinned = dec.pinned_input(batch, params.n_c)
        pinned[:] = blocks
        res = dec.decode(pinned)
    finally:
        dec.close()
    ref = nr.decode(blocks, bg, cfg)
    assert np.array_equal(res.bits, ref.bits) and np.array_equal(res.iterations, ref.iterations)
    assert np.array_equal(res.syndrome_weight, ref.syndrome_weight) and np.array_equal(res.success, ref.success)
    if stop == "crc":
        assert np.array_equal(res.crc_ok, ref.crc_ok)


@pytest.mark.parametrize("prec,bg_id,z,rows,stop,batch", [
    ("f16", "BG1", 384, 46, "none", 33), ("f32", "BG1", 384, 46, "syndrome", 17),
    ("f16", "BG2", 384, 42, "syndrome", 40), ("f32", "BG2", 256, 20, "none", 9),
    ("f16", "BG1", 288, 9, "none", 5), ("f16", "BG1", 384, 4, "syndrome", 4)])
def test_float_on_chip_messages_match_workspace_and_oracle(cuda_ok, prec, bg_id, z, rows, stop, batch, monkeypatch):
    """Single-group BG1/BG2 float shapes keep their messages on chip (shared
    and tensor memory; BG1 core rows in the workspace); NRLDPC_NO_TM=1 keeps
    them all in the global workspace. Both must give the oracle's results."""
    monkeypatch.delenv("NRLDPC_NO_TM", raising=False)  # the first plan must keep messages on chip
    bg = nr.load_basegraph(bg_id, z)
    params = nr.code_params(bg, z, rows)
    _, llr = noisy_llrs(bg, rows, 1.5, batch, seed=(z, rows, 5))
    blocks = nr.quantize(llr, nr.QuantConfig(mode=prec), params)
    cfg = nr.DecodeConfig(max_iter=7, early_stop=stop, precision=prec)
    ref = oracle.decode(blocks, bg, cfg)
    smem = []
    for no_tm in (False, True):
        if no_tm:
            monkeypatch.setenv("NRLDPC_NO_TM", "1")
        plan = nr.Plan(bg, rows, cfg)
        smem.append(plan.smem_bytes)
        out = plan.alloc_outputs(batch)
        plan.decode_device(torch.from_numpy(blocks).cuda(), out)
        torch.cuda.synchronize()
        assert np.array_equal(nr.unpack_bits(out["bits"].cpu().numpy(), params.k), ref["bits"])
        assert np.array_equal(out["iters"].cpu().numpy(), ref["iterations"])
        assert np.array_equal(out["synd"].cpu().numpy(), ref["syndrome_weight"])
    assert smem[0] != smem[1]


def test_tm_plans_concurrent_with_each_other_and_cublas(cuda_ok):
    """TM-layout kernels allocate all 512 tensor-memory columns of their SM.
    Several TM plans on concurrent streams, next to cuBLAS GEMMs (which use
    tensor memory on sm_100) on another stream, must neither deadlock nor
    change results."""
    cases = [("BG1", 384, 46), ("BG2", 384, 42), ("BG1", 256, 46), ("BG1", 320, 30)]
    plans, blocks, refs, outs = [], [], [], []
    for bg_id, z, rows in cases:
        bg = nr.load_basegraph(bg_id, z)
        cfg = nr.DecodeConfig(max_iter=6, early_stop="syndrome")
        _, llr = noisy_llrs(bg, rows, 1.5, 150, seed=(z, rows, 3))
        b = oracle.quantize_i8(llr, z)
        plans.append(nr.Plan(bg, rows, cfg))
        blocks.append(torch.from_numpy(b).cuda())
        refs.append(oracle.decode(b, bg, cfg))
        outs.append([plans[-1].alloc_outputs(150) for _ in range(3)])
    streams = [torch.cuda.Stream() for _ in range(len(cases))]
    gemm_stream = torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()
    with torch.cuda.stream(gemm_stream):
        for _ in range(8):
            a = (a @ a).clamp_(-1, 1)
    for rep in range(3):
        for i, plan in enumerate(plans):
            plan.decode_device(blocks[i], outs[i][rep], stream=streams[i].cuda_stream)
    torch.cuda.synchronize()
    for i, (bg_id, z, rows) in enumerate(cases):
        k = nr.code_params(nr.load_basegraph(bg_id, z), z, rows).k
        for rep in range(3):
            o = outs[i][rep]
            assert np.array_equal(nr.unpack_bits(o["bits"].cpu().numpy(), k), refs[i]["bits"])
            assert np.array_equal(o["iters"].cpu().numpy(), refs[i]["iterations"])
