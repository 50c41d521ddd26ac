"""Freeze golden decode vectors from the REFERENCE implementation.

Runs only in the build container, where /root/reference exists:
    python tests/golden/make_golden.py
It imports ldpclab (the reference package) and the reference's own test
fixture generator ``tests.conftest.make_noisy_blocks`` in place, decodes each
case with ``ldpclab.decoder.decode`` and stores inputs + outputs in
``tests/golden/golden.npz`` (+ ``cases.json``). The GPU box has no
/root/reference; tests there compare the CUDA path against these files and
against the C oracle (which these files pin).
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF)]
sys.dont_write_bytecode = True

from ldpclab import basegraph as rbg  # noqa: E402
from ldpclab import channel as rch  # noqa: E402
from ldpclab import codec as rcodec  # noqa: E402
from ldpclab import decoder as rdec  # noqa: E402
from tests.conftest import make_noisy_blocks  # noqa: E402  (reference fixture)

OUT = Path(__file__).resolve().parent
CASES = []


def case(name, bg_id, z, rows, blocks, **cfg_kw):
    trace_on = cfg_kw.pop("trace", False)
    flooding = cfg_kw.pop("flooding", False)
    cfg = rdec.DecodeConfig(**cfg_kw)
    bg = rbg.load_basegraph(bg_id, z)
    trace = [] if trace_on else None
    res = (rdec.decode_flooding if flooding else rdec.decode)(blocks, bg, cfg, trace)
    meta = {"name": name, "bg": bg_id, "z": z, "rows": rows, "trace": trace_on, "flooding": flooding,
            "cfg": {k: (v.value if hasattr(v, "value") else v) for k, v in cfg.__dict__.items()}}
    arrays = {
        "llr": np.asarray(blocks),
        "bits": np.packbits(res.bits, axis=1, bitorder="little"),
        "iterations": res.iterations.astype(np.int64),
        "success": res.success.astype(np.uint8),
        "syndrome_weight": res.syndrome_weight.astype(np.int64),
    }
    if res.crc_ok is not None:
        arrays["crc_ok"] = res.crc_ok.astype(np.uint8)
    if trace is not None:
        arrays["trace"] = np.array([[c, i, w, m] for c, i, w, m in trace], dtype=np.float64)
    CASES.append((meta, arrays))
    print(f"{name}: B={len(res.iterations)} iters={res.iterations.min()}..{res.iterations.max()} "
          f"success={res.success.mean():.2f}", flush=True)


def crc_blocks(bg, rows, ebn0, count, seed, kind="crc24b"):
    params = rbg.code_params(bg, bg.z, rows)
    rng = np.random.default_rng(seed)
    length = rcodec.CRC_POLYS[kind][0]
    payload = rng.integers(0, 2, size=(count, params.k - length), dtype=np.uint8)
    msgs = np.stack([rcodec.crc_attach(p, kind, k=params.k) for p in payload])
    tx = rcodec.encode_batch(msgs, bg, bg.z, rows)[:, 2 * bg.z:]
    sigma = rch.ebn0_to_sigma(ebn0, params.k / params.n_tx)
    llr = rch.demap_llr(rch.bpsk_awgn(tx, sigma, rng), sigma)
    return rch.quantize(llr, rch.QuantConfig(), params)


def noise_free(bg, rows, seed, mode="int8", mag=16.0):
    params = rbg.code_params(bg, bg.z, rows)
    rng = np.random.default_rng(seed)
    msg = rng.integers(0, 2, params.k, dtype=np.uint8)
    cw = rcodec.encode(msg, bg, bg.z, rows)
    llr = rch.bpsk_exact(rcodec.puncture(cw)) * mag
    return rch.quantize(llr, rch.QuantConfig(mode=mode), params)[None, :]


def main():
    g = rbg.load_basegraph
    I8 = rdec.Precision.INT8
    # --- BASELINE.json configs ------------------------------------------------
    # config 1: harness.run_latency_bench input (seed (0,0), 4 dB), 10 fixed iterations
    bg = g("BG2", 64)
    params = rbg.code_params(bg, 64, 42)
    rng = np.random.default_rng((0, 0))
    msgs = rng.integers(0, 2, size=(4, params.k), dtype=np.uint8)
    tx = rcodec.encode_batch(msgs, bg, 64, 42)[:, 128:]
    sigma = rch.ebn0_to_sigma(4.0, params.k / params.n_tx)
    blk = rch.quantize(rch.demap_llr(rch.bpsk_awgn(tx, sigma, rng), sigma), rch.QuantConfig(), params)
    case("cfg1_bg2_z64_none10", "BG2", 64, 42, blk, precision=I8, max_iter=10,
         early_stop="none")
    # config 2: headline shape, fixed 10 iterations
    _, blk = make_noisy_blocks(g("BG1", 384), 46, 2.0, 6, seed=2024)
    case("cfg2_bg1_z384_none10", "BG1", 384, 46, blk, precision=I8, max_iter=10, early_stop="none")
    # config 3: low SNR, syndrome early termination
    _, blk = make_noisy_blocks(g("BG2", 384), 42, 0.5, 6, seed=3)
    case("cfg3_bg2_z384_syn20", "BG2", 384, 42, blk, precision=I8, max_iter=20)
    # --- small graphs, every stop mode ------------------------------------------
    _, blk = make_noisy_blocks(g("BG2", 16), 42, 1.5, 64, seed=7)
    case("bg2_z16_syn12", "BG2", 16, 42, blk, precision=I8, max_iter=12)
    case("bg2_z16_none10", "BG2", 16, 42, blk, precision=I8, max_iter=10, early_stop="none")
    case("bg2_z16_ll_alpha4", "BG2", 16, 42, blk, precision=I8, max_iter=12,
         strategy="low_latency", alpha=4)
    case("bg2_z16_rho4", "BG2", 16, 42, blk, precision=I8, max_iter=12, rho=4)
    _, blk = make_noisy_blocks(g("BG2", 16), 42, 2.0, 8, seed=43)
    case("bg2_z16_trace", "BG2", 16, 42, blk, precision=I8, max_iter=6, trace=True)
    case("bg2_z16_rho4_trace", "BG2", 16, 42, blk, precision=I8, max_iter=8, rho=4, trace=True)
    case("bg2_z16_none_trace", "BG2", 16, 42, blk, precision=I8, max_iter=5, early_stop="none",
         trace=True)
    blk = crc_blocks(g("BG2", 16), 42, 1.75, 32, seed=(808, 1, 0))
    case("bg2_z16_crc", "BG2", 16, 42, blk, precision=I8, max_iter=20, early_stop="crc")
    blk = crc_blocks(g("BG2", 32), 42, 1.75, 16, seed=(808, 2, 0), kind="crc16")
    case("bg2_z32_crc16", "BG2", 32, 42, blk, precision=I8, max_iter=20, early_stop="crc",
         crc_kind="crc16")
    blk = noise_free(g("BG2", 16), 42, 41)  # valid codeword, payload fails CRC
    case("bg2_z16_crc_reject", "BG2", 16, 42, blk, precision=I8, max_iter=5, early_stop="crc")
    # beta: default LUT path plus non-dyadic values
    _, blk = make_noisy_blocks(g("BG2", 32), 42, 1.5, 32, seed=11)
    for beta in (0.5, 1.0, 0.8, 0.6875):
        case(f"bg2_z32_beta{beta}", "BG2", 32, 42, blk, precision=I8, max_iter=15, beta=beta)
    # partial rows (higher rate), both graphs
    _, blk = make_noisy_blocks(g("BG2", 16), 10, 2.5, 16, seed=59)
    case("bg2_z16_rows10", "BG2", 16, 10, blk, precision=I8, max_iter=20)
    _, blk = make_noisy_blocks(g("BG1", 8), 8, 3.0, 16, seed=60)
    case("bg1_z8_rows8", "BG1", 8, 8, blk, precision=I8, max_iter=20)
    _, blk = make_noisy_blocks(g("BG1", 384), 8, 3.0, 4, seed=61)
    case("bg1_z384_rows8", "BG1", 384, 8, blk, precision=I8, max_iter=20)
    # odd / small Z (several codewords per warp on the GPU)
    for bg_id, z, rows in (("BG1", 2, 46), ("BG1", 3, 46), ("BG2", 5, 42), ("BG1", 7, 46),
                           ("BG2", 9, 42), ("BG1", 11, 46), ("BG2", 13, 42), ("BG1", 15, 46),
                           ("BG1", 52, 46), ("BG2", 104, 42), ("BG1", 208, 46), ("BG2", 240, 42),
                           ("BG1", 288, 46), ("BG1", 352, 46)):
        _, blk = make_noisy_blocks(g(bg_id, z), rows, 2.0, 8 if z < 200 else 4, seed=(z, rows))
        case(f"{bg_id.lower()}_z{z}_syn20", bg_id, z, rows, blk, precision=I8, max_iter=20)
    # total erasure (decoder fixed point) and noise-free round trips
    case("bg2_z16_erasure", "BG2", 16, 42, np.zeros((2, 832), np.int8), precision=I8, max_iter=7)
    for bg_id in ("BG1", "BG2"):
        for z in (2, 16, 384):
            blk = noise_free(g(bg_id, z), g(bg_id, z).m_bg, (6, z))
            case(f"{bg_id.lower()}_z{z}_noisefree", bg_id, z, g(bg_id, z).m_bg, blk, precision=I8)
    # float precisions (next §8 row; pins the oracle now)
    _, blk = make_noisy_blocks(g("BG2", 16), 42, 2.0, 16, seed=47, mode="f32")
    case("bg2_z16_f32", "BG2", 16, 42, blk, precision="f32", max_iter=20)
    case("bg2_z16_f32_trace", "BG2", 16, 42, blk[:4], precision="f32", max_iter=6, trace=True)
    _, blk = make_noisy_blocks(g("BG2", 16), 42, 2.0, 16, seed=48, mode="f16")
    case("bg2_z16_f16", "BG2", 16, 42, blk, precision="f16", max_iter=20)
    _, blk = make_noisy_blocks(g("BG1", 32), 46, 1.75, 8, seed=49, mode="f16")
    case("bg1_z32_f16_none", "BG1", 32, 46, blk, precision="f16", max_iter=10, early_stop="none")
    # flooding schedule (decoder.py:337-365, 569-581)
    _, blk = make_noisy_blocks(g("BG2", 16), 42, 2.5, 24, seed=29, mode="f32")
    case("flood_bg2_z16_f32", "BG2", 16, 42, blk, precision="f32", max_iter=50, flooding=True)
    case("flood_bg2_z16_f32_trace", "BG2", 16, 42, blk[:4], precision="f32", max_iter=8,
         flooding=True, trace=True)
    _, blk = make_noisy_blocks(g("BG2", 16), 42, 2.0, 24, seed=30)
    case("flood_bg2_z16_i8", "BG2", 16, 42, blk, precision=I8, max_iter=20, flooding=True)
    case("flood_bg2_z16_i8_none", "BG2", 16, 42, blk, precision=I8, max_iter=6, flooding=True,
         early_stop="none")
    _, blk = make_noisy_blocks(g("BG1", 24), 46, 2.0, 8, seed=31, mode="f16")
    case("flood_bg1_z24_f16", "BG1", 24, 46, blk, precision="f16", max_iter=20, flooding=True)
    _, blk = make_noisy_blocks(g("BG1", 104), 10, 3.0, 8, seed=32)
    case("flood_bg1_z104_rows10_i8", "BG1", 104, 10, blk, precision=I8, max_iter=15, flooding=True)
    blk = noise_free(g("BG2", 16), 42, 19, mode="f32")
    case("flood_bg2_z16_noisefree", "BG2", 16, 42, blk, precision="f32", flooding=True)
    # config 4 shape: every lifting size, both graphs, 2 codewords each
    for bg_id in ("BG1", "BG2"):
        for z in rbg.ALL_LIFTING_SIZES:
            bgz = g(bg_id, z)
            _, blk = make_noisy_blocks(bgz, bgz.m_bg, 2.0, 2, seed=(int(bg_id[-1]), z))
            case(f"sweep_{bg_id.lower()}_z{z}", bg_id, z, bgz.m_bg, blk, precision=I8, max_iter=10,
                 early_stop="none")

    # quantizer vectors (channel.quantize): ties at .5 steps, clipping, punctures
    qz = []
    params = rbg.code_params(g("BG2", 16), 16, 42)
    rng = np.random.default_rng(99)
    x = rng.normal(0, 8, size=(3, params.n_tx))
    x[0, :16] = (np.arange(16) - 8) / 8.0 + 1 / 16.0      # exact .5 ties after *8
    x[1, :4] = [1e6, -1e6, 15.9375, -15.9375]
    for mode in ("int8", "f16", "f32"):
        q = rch.quantize(x, rch.QuantConfig(mode=mode), params)
        qz.append((mode, q))

    arrays = {}
    metas = []
    for meta, arr in CASES:
        metas.append(meta)
        for k, v in arr.items():
            arrays[f"{meta['name']}/{k}"] = v
    arrays["quant/x"] = x
    for mode, q in qz:
        arrays[f"quant/{mode}"] = q
    np.savez_compressed(OUT / "golden.npz", **arrays)
    prov = {"cases": metas,
            "reference": "ldpclab 0.1.0 at /root/reference/pkg (decoder.decode, channel.quantize)",
            "assets_sha256": json.loads((REF / "src/ldpclab/assets/manifest.json").read_text())}
    (OUT / "cases.json").write_text(json.dumps(prov, indent=1) + "\n")
    h = hashlib.sha256((OUT / "golden.npz").read_bytes()).hexdigest()
    print("wrote", OUT / "golden.npz", (OUT / "golden.npz").stat().st_size, "bytes sha256", h)


if __name__ == "__main__":
    main()
