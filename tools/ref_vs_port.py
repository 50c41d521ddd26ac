"""CPU baseline cross-check (run in the survey container, where /root/reference
exists): the reference's own numpy decoder vs the C port (oracle/) on the
same codewords, one core each, bit-exact outputs compared. The GPU box has no
/root/reference, so bench.py's CPU arm times the port; this records how the
port relates to the reference itself."""
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

import ldpclab  # noqa: E402
from oracle import oracle  # noqa: E402
import paper_2009_05534_b200 as nr  # noqa: E402
from paper_2009_05534_b200.synth import noisy_llrs  # noqa: E402

print(f"host: {os.cpu_count()} cpus; numpy {np.__version__}")
for bg_id, z, rows, n in (("BG1", 384, 46, 8), ("BG2", 384, 42, 8), ("BG2", 64, 42, 16)):
    bg = nr.load_basegraph(bg_id, z)
    _, llr = noisy_llrs(bg, rows, 2.0, n, seed=(7, z))
    blocks = oracle.quantize_i8(llr, z)
    rbg = ldpclab.load_basegraph(int(bg_id[-1]), z)
    rcfg = ldpclab.DecodeConfig(max_iter=10, early_stop="none")
    ref_decode = ldpclab.decode
    ref_decode(blocks[:1], rbg, rcfg)
    t0 = time.perf_counter()
    ref = ref_decode(blocks, rbg, rcfg)
    t_ref = time.perf_counter() - t0
    cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
    t0 = time.perf_counter()
    port = oracle.decode(blocks, bg, cfg, threads=1)
    t_port = time.perf_counter() - t0
    same = np.array_equal(ref.bits, port["bits"]) and np.array_equal(ref.iterations, port["iterations"])
    k = bg.k_b * z
    print(f"{bg_id} Z={z} rows={rows}, {n} codewords, 10 iterations, 1 core: reference numpy "
          f"{n * k / t_ref / 1e6:.3f} Mbps, C port {n * k / t_port / 1e6:.3f} Mbps "
          f"(port / reference = {t_ref / t_port:.1f}x), outputs bit-exact: {same}")
