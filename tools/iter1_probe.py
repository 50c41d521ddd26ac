#!/usr/bin/env python
"""One decode launch at 1 fixed iteration (BG1 Z=384, one wave of 296
codewords) for profiling the per-CTA fixed cost (tools/iter_probe.py)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import torch  # noqa: E402

import paper_2009_05534_b200 as nr  # noqa: E402
from bench_configs import gpu_blocks  # noqa: E402

bg = nr.load_basegraph(1, 384)
_, blocks = gpu_blocks(bg, 46, 2.0, 296, 1)
plan = nr.Plan(bg, 46, nr.DecodeConfig(max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 1, early_stop="none"))
out = plan.alloc_outputs(296)
for _ in range(3):
    plan.decode_device(blocks, out)
torch.cuda.synchronize()
