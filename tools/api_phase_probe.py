"""Where the reference-facing decode(numpy) time goes (BG1 Z=384, B=1024)."""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2009_05534_b200 as nr  # noqa: E402
from paper_2009_05534_b200.decoder import unpack_bits  # noqa: E402


def t(fn, n=10):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e3


print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
bg = nr.load_basegraph("BG1", 384)
cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
plan = nr.get_plan(bg, 46, cfg)
rng = np.random.default_rng(0)
x = rng.integers(-127, 128, size=(1024, plan.n_c), dtype=np.int8)
pin = torch.empty(x.shape, dtype=torch.int8, pin_memory=True).numpy()
pin[:] = x
print("np.copyto 26.7MB pageable->pinned (1 thread) ms", t(lambda: np.copyto(pin, x)))
print("np.empty+fill 8.6MB ms", t(lambda: np.empty((1024, 8448), np.uint8).fill(1)))
hout = plan.host_outputs(1024, pinned=True)
pout = plan.host_outputs(1024, pinned=False)
print("decode_host pinned in, pinned out ms", t(lambda: plan.decode_host(pin, chunks=12, out=hout)))
print("decode_host pageable in, pinned out ms", t(lambda: plan.decode_host(x, chunks=12, out=hout)))
print("decode_host pageable in, pageable out ms", t(lambda: plan.decode_host(x, chunks=12, out=pout)))
for ch in (4, 8, 24):
    print(f"  chunks={ch} pageable/pageable ms", t(lambda: plan.decode_host(x, chunks=ch, out=pout)))
print("unpack_bits ms", t(lambda: unpack_bits(pout["bits"], plan.k)))
print("nr.decode(numpy) ms", t(lambda: nr.decode(x, bg, cfg)))
