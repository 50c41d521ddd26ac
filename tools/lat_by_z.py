#!/usr/bin/env python
"""Per-Z decode latency of small batches (the mixed-batch config's launches).

    python tools/lat_by_z.py [batch] [so_path]
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
if len(sys.argv) > 2:
    os.environ["NRLDPC_LIB"] = sys.argv[2]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_05534_b200 as nr  # noqa: E402
sys.path.insert(0, str(ROOT / "tools"))
from bench_configs import gpu_blocks, time_plan  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 16
res = {}
for bgn in (1, 2):
    for z in (64, 128, 192, 224, 256, 288, 320, 352, 384):
        bg = nr.load_basegraph(bgn, z)
        cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
        plan = nr.Plan(bg, bg.m_bg, cfg)
        _, blocks = gpu_blocks(bg, bg.m_bg, 2.0, batch, 1)
        out = plan.alloc_outputs(batch)
        t = time_plan(plan, blocks, out, 30)
        res[f"bg{bgn}_z{z}"] = round(float(np.median(t)) * 1e3, 1)
print(json.dumps(res))
