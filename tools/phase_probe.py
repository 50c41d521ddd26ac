"""Per-CTA phase durations of the headline kernel (BG1 Z=384, one wave of
148 pair-CTAs, 10 iterations) from a NRLDPC_PHASES build:
  make -C paper_2009_05534_b200/csrc phases
  NRLDPC_LIB=paper_2009_05534_b200/libnrldpc_phases.so python tools/phase_probe.py"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import paper_2009_05534_b200 as nr  # noqa: E402
from paper_2009_05534_b200 import _native  # noqa: E402
from bench_configs import gpu_blocks  # noqa: E402

bg = nr.load_basegraph("BG1", 384)
ctas = torch.cuda.get_device_properties(0).multi_processor_count
B = 2 * ctas * int(sys.argv[1]) if len(sys.argv) > 1 else 2 * ctas
_, blocks = gpu_blocks(bg, 46, 2.0, B, (2024, 0))
plan = nr.Plan(bg, 46, nr.DecodeConfig(max_iter=10, early_stop="none"))
out = plan.alloc_outputs(B)
for _ in range(3):
    plan.decode_device(blocks, out)
torch.cuda.synchronize()
lib = _native.load()
n = B // 2
buf = (ctypes.c_ulonglong * (n * 16))()
lib.nrldpc_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert lib.nrldpc_debug_phases(buf, n * 16) == 0
t8 = np.array(buf, dtype=np.float64).reshape(n, 16) / 1e3  # us
t = t8[:, :5]
d = np.diff(t, axis=1)
names = ["prologue", "10 iterations", "final check + results", "TMEM dealloc/exit"]
for i, nm in enumerate(names):
    print(f"{nm:24s} median {np.median(d[:, i]):8.2f} us   p10 {np.percentile(d[:, i], 10):8.2f}  p90 {np.percentile(d[:, i], 90):8.2f}")
sub = np.stack([t8[:, 5] - t8[:, 2], t8[:, 6] - t8[:, 5], t8[:, 7] - t8[:, 6], t8[:, 3] - t8[:, 7]], axis=1)
for i, nm in enumerate(["  parity + margin scan", "  counters + barrier", "  bit packing", "  result words + barriers"]):
    print(f"{nm:24s} median {np.median(sub[:, i]):8.2f} us")
print(f"CTA total median {np.median(t[:, 4] - t[:, 0]):.2f} us; first entry to last exit {t[:, 4].max() - t[:, 0].min():.2f} us")
if t8[:, 8].any():  # bit-sliced final check (pack_hard_tm / packed_parity_tm)
    for nm, a, b in (("    barrier after the last layer", 2, 8), ("    pack (hard words + margin)", 8, 9),
                     ("    barrier", 9, 10), ("    packed parity", 10, 5)):
        print(f"{nm:34s} median {np.median(t8[:, b] - t8[:, a]):8.2f} us")
