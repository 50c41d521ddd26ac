"""Randomized differential test on the GPU: many (graph, Z, rows_used, beta,
stop mode, precision, batch) combinations against the oracle. Every kernel
variant the shape chooser can pick is reached: pair / single lanes, register
rows, absolute or relative addressing, paired message words, lane refill,
generic schedule (table-only betas), float engines."""

import os

import numpy as np
import pytest

import paper_2009_05534_b200 as nr
from paper_2009_05534_b200.synth import noisy_llrs
from oracle import oracle

pytestmark = pytest.mark.gpu

ZS = nr.ALL_LIFTING_SIZES


FUZZ_N = int(os.environ.get("NRLDPC_FUZZ_N", "100"))
FUZZ_SEED = int(os.environ.get("NRLDPC_FUZZ_SEED", "20260"))


def _cases(n=FUZZ_N, seed=FUZZ_SEED):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        bg_id = "BG1" if rng.random() < 0.55 else "BG2"
        z = int(rng.choice(ZS))
        m_bg = 46 if bg_id == "BG1" else 42
        rows = int(rng.choice([4, 5, 6, 7, 8, 12, m_bg, m_bg, m_bg]))
        rows = min(rows, m_bg)
        beta = float(rng.choice([0.75, 0.75, 0.5, 0.8, 0.625, 0.3, 0.7, 1.0]))
        stop = str(rng.choice(["none", "syndrome", "syndrome", "crc"]))
        prec = str(rng.choice(["int8", "int8", "int8", "f16", "f32"]))
        batch = int(rng.choice([1, 2, 3, 7, 16, 33, 130]))
        ebn0 = float(rng.uniform(0.5, 3.5))
        out.append((i, bg_id, z, rows, beta, stop, prec, batch, ebn0))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c[0]}-{c[1]}-z{c[2]}-r{c[3]}-{c[6]}-{c[5]}")
def test_fuzz_vs_oracle(cuda_ok, case):
    i, bg_id, z, rows, beta, stop, prec, batch, ebn0 = case
    bg = nr.load_basegraph(bg_id, z)
    params = nr.code_params(bg, z, rows)
    if stop == "crc" and params.k <= 24:
        stop = "syndrome"
    _, llr = noisy_llrs(bg, rows, ebn0, batch, seed=(i, z, rows))
    qc = nr.QuantConfig(mode=prec)
    blocks = nr.quantize(llr, qc, params)
    cfg = nr.DecodeConfig(max_iter=int(3 + i % 9), beta=beta, early_stop=stop, precision=prec)
    ref = oracle.decode(blocks, bg, cfg)
    res = nr.decode(blocks, bg, cfg)
    bad = np.flatnonzero((res.bits != ref["bits"]).any(axis=1))
    assert bad.size == 0, f"bits differ in codewords {bad[:8]}"
    assert np.array_equal(res.iterations, ref["iterations"])
    assert np.array_equal(res.success, ref["success"])
    assert np.array_equal(res.syndrome_weight, ref["syndrome_weight"])
    if stop == "crc":
        assert np.array_equal(res.crc_ok, ref["crc_ok"])


def _tm_cases(n=max(1, FUZZ_N // 2), seed=FUZZ_SEED + 1):
    """Shapes that decode on the TM layout (single-group pairs holding an SM
    alone: BG1 Z = 160..384, BG2 Z = 256..384, multiples of 32)."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        bg_id = "BG1" if rng.random() < 0.6 else "BG2"
        z = int(rng.choice([160, 192, 224, 256, 288, 320, 352, 384] if bg_id == "BG1" else [256, 288, 320, 352, 384]))
        m_bg = 46 if bg_id == "BG1" else 42
        rows = int(rng.choice([6, 7, 9, 17, 30, m_bg, m_bg]))
        stop = str(rng.choice(["none", "syndrome", "syndrome", "crc"]))
        batch = int(rng.choice([1, 2, 3, 5, 40, 301]))
        out.append((i, bg_id, z, rows, stop, batch, float(rng.uniform(0.5, 3.0))))
    return out


@pytest.mark.parametrize("case", _tm_cases(), ids=lambda c: f"tm{c[0]}-{c[1]}-z{c[2]}-r{c[3]}-{c[4]}-b{c[5]}")
def test_fuzz_tm_shapes_vs_oracle(cuda_ok, case):
    i, bg_id, z, rows, stop, batch, ebn0 = case
    bg = nr.load_basegraph(bg_id, z)
    params = nr.code_params(bg, z, rows)
    _, llr = noisy_llrs(bg, rows, ebn0, batch, seed=(i, z, rows, 7))
    blocks = nr.quantize(llr, nr.QuantConfig(), params)
    cfg = nr.DecodeConfig(max_iter=int(4 + i % 12), early_stop=stop)
    ref = oracle.decode(blocks, bg, cfg)
    res = nr.decode(blocks, bg, cfg)
    bad = np.flatnonzero((res.bits != ref["bits"]).any(axis=1))
    assert bad.size == 0, f"bits differ in codewords {bad[:8]}"
    assert np.array_equal(res.iterations, ref["iterations"])
    assert np.array_equal(res.success, ref["success"])
    assert np.array_equal(res.syndrome_weight, ref["syndrome_weight"])
    if stop == "crc":
        assert np.array_equal(res.crc_ok, ref["crc_ok"])
