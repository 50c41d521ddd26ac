"""Wall-clock of the reference-facing Python API (host numpy in, DecodeResult out)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2009_05534_b200 as nr  # noqa: E402
from paper_2009_05534_b200.synth import noisy_llrs  # noqa: E402
from oracle import oracle  # noqa: E402

for bgn, z, B in ((1, 384, 1024), (2, 64, 1), (1, 384, 16)):
    bg = nr.load_basegraph(bgn, z)
    rows = bg.m_bg
    _, llr = noisy_llrs(bg, rows, 2.0, min(B, 64), seed=1)
    blk = oracle.quantize_i8(llr, z)
    blk = np.concatenate([blk] * (B // len(blk) + 1))[:B]
    cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
    for _ in range(3):
        nr.decode(blk, bg, cfg)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        nr.decode(blk, bg, cfg)
        ts.append(time.perf_counter() - t0)
    print(f"BG{bgn} Z={z} B={B}: nr.decode p50 {np.median(ts) * 1e3:.2f} ms")
