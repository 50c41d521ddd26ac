#!/usr/bin/env python
"""A/B two plan-creation environments in one process, timed alternately.

    python tools/ab_env.py VAR=VALUE [batch]   (A: VAR unset, B: VAR set)
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import paper_2009_05534_b200 as nr  # noqa: E402
from bench_configs import gpu_blocks, time_plan  # noqa: E402

var, val = sys.argv[1].split("=", 1)
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cases = [(1, 64), (1, 192), (1, 256), (1, 288), (1, 384), (2, 128), (2, 256), (2, 384)]
cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
for bgn, z in cases:
    bg = nr.load_basegraph(bgn, z)
    _, blocks = gpu_blocks(bg, bg.m_bg, 2.0, batch, 1)
    os.environ.pop(var, None)
    pa = nr.Plan(bg, bg.m_bg, cfg)
    os.environ[var] = val
    pb = nr.Plan(bg, bg.m_bg, cfg)
    os.environ.pop(var, None)
    oa, ob = pa.alloc_outputs(batch), pb.alloc_outputs(batch)
    ta, tb = [], []
    for _ in range(5):
        ta += list(time_plan(pa, blocks, oa, 20))
        tb += list(time_plan(pb, blocks, ob, 20))
    same = torch.equal(oa["bits"], ob["bits"])
    shp = lambda q: (q.lanes, q.groups_per_cta, q.threads_per_cta, q.smem_bytes)
    if shp(pa) != shp(pb):
        print("  shapes differ:", shp(pa), shp(pb))
    print(f"bg{bgn} z{z} B={batch}: A {np.median(ta) * 1e3:8.1f} us  B({var}) {np.median(tb) * 1e3:8.1f} us  "
          f"B/A {np.median(tb) / np.median(ta):.3f} same={same}")
