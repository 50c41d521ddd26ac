#!/usr/bin/env python
"""Randomized parity sweep of the CUDA decoder against the oracle.

Draws random (graph, Z, rows_used, batch, Eb/N0, precision, stop mode,
max_iter, beta) cases for a time budget, decodes each through the public
`decode` and through the oracle (oracle/, the CPU restatement pinned to the
reference's golden vectors), and reports every mismatch. A companion to the
fixed-case GPU tests: it walks the shape space (all 51 Z, partial graphs,
odd batches) the fixed cases only sample. One case in ten is a random mixed
batch through MixedBatchDecoder (multi-shape launches in a CUDA graph), and
about one in seven single-shape cases also compares the per-iteration trace.

    python tools/parity_sweep.py [seconds=240] [seed=0]
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2009_05534_b200 as nr  # noqa: E402
from paper_2009_05534_b200.synth import noisy_llrs  # noqa: E402
from oracle import oracle  # noqa: E402


def case(rng):
    bg_id = "BG1" if rng.random() < 0.5 else "BG2"
    z = int(rng.choice(nr.ALL_LIFTING_SIZES))
    bg = nr.load_basegraph(bg_id, z)
    rows = int(bg.m_bg if rng.random() < 0.6 else rng.integers(4, bg.m_bg + 1))
    big = z * bg.n_cols >= 8000
    batch = int(rng.integers(1, 9 if big else 40))
    prec = str(rng.choice(["int8"] * 6 + ["f16", "f32"]))
    stop = str(rng.choice(["none", "syndrome", "crc"]))
    if stop == "crc" and bg.k_b * z < 40:
        stop = "syndrome"  # too few bits for a CRC field
    cfg = nr.DecodeConfig(precision=prec, early_stop=stop, max_iter=int(rng.integers(1, 13)),
                          beta=float(rng.choice([0.75, 0.5, 0.625, 0.875, 1.0])))
    ebn0 = float(rng.uniform(-1.0, 4.0))
    return bg, rows, batch, cfg, ebn0


def mixed_case(rng, seed, n):
    """A random mixed batch (MixedBatchDecoder: multi-shape launches in one
    CUDA-graph replay) of 2..12 int8 groups, each group against the oracle."""
    from paper_2009_05534_b200.mixed import Group, MixedBatchDecoder
    stop = str(rng.choice(["none", "syndrome", "crc"]))
    cfg = nr.DecodeConfig(early_stop=stop, max_iter=int(rng.integers(1, 11)))
    groups, data = [], []
    for g in range(int(rng.integers(2, 13))):
        bg = nr.load_basegraph("BG1" if rng.random() < 0.5 else "BG2", int(rng.choice(nr.ALL_LIFTING_SIZES)))
        if stop == "crc" and bg.k_b * bg.z < 40:
            bg = nr.load_basegraph(bg.id, 384)
        rows = int(bg.m_bg if rng.random() < 0.7 else rng.integers(4, bg.m_bg + 1))
        batch = int(rng.integers(1, 12))
        _, llr = noisy_llrs(bg, rows, float(rng.uniform(-1.0, 4.0)), batch, seed=(seed, n, g))
        groups.append(Group(bg, rows, batch))
        data.append(oracle.quantize_i8(llr, bg.z))
    mixed = MixedBatchDecoder(groups, cfg, streams=int(rng.integers(1, 9)), grouped=bool(rng.random() < 0.8))
    ok, cws = True, 0
    for res, g, blocks in zip(mixed.decode(data), groups, data):
        ref = oracle.decode(blocks, g.bg, cfg)
        ok = ok and np.array_equal(res.bits, ref["bits"]) and np.array_equal(res.iterations, ref["iterations"]) \
            and np.array_equal(res.success, ref["success"]) \
            and np.array_equal(res.syndrome_weight, ref["syndrome_weight"])
        cws += g.batch
    if not ok:
        print(f"MISMATCH mixed batch {[(g.bg.id, g.bg.z, g.rows_used, g.batch) for g in groups]} {cfg}", flush=True)
    return ok, cws


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rng = np.random.default_rng(seed)
    t0 = time.time()
    n = bad = cw = 0
    while time.time() - t0 < budget:
        if rng.random() < 0.1:  # one case in ten is a mixed batch
            ok, c = mixed_case(rng, seed, n)
            bad += 0 if ok else 1
            n += 1
            cw += c
            continue
        bg, rows, batch, cfg, ebn0 = case(rng)
        _, llr = noisy_llrs(bg, rows, ebn0, batch, seed=(seed, n))
        if cfg.precision.value == "int8":
            blocks = oracle.quantize_i8(llr, bg.z)
        else:
            dt = np.float16 if cfg.precision.value == "f16" else np.float32
            blocks = np.concatenate([np.zeros((batch, 2 * bg.z)), llr], axis=1).astype(dt)
        traced = rng.random() < 0.15  # per-iteration (codeword, iteration, weight, margin) trace
        tr_ref, tr = ([], []) if traced else (None, None)
        ref = oracle.decode(blocks, bg, cfg, tr_ref)
        got = nr.decode(blocks, bg, cfg, tr)
        ok = (tr == tr_ref and np.array_equal(got.bits, ref["bits"]) and np.array_equal(got.iterations, ref["iterations"])
              and np.array_equal(got.success, ref["success"])
              and np.array_equal(got.syndrome_weight, ref["syndrome_weight"]))
        if cfg.early_stop.value == "crc":
            ok = ok and np.array_equal(got.crc_ok, ref["crc_ok"])
        if not ok:
            bad += 1
            print(f"MISMATCH {bg.id} Z={bg.z} rows={rows} B={batch} {cfg} ebn0={ebn0:.2f}", flush=True)
        n += 1
        cw += batch
    print(f"{n} cases, {cw} codewords, {bad} mismatches in {time.time() - t0:.0f} s (seed {seed})")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
