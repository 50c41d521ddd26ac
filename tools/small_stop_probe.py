#!/usr/bin/env python
"""Early-stop (syndrome, max 20) batch time for byte-pair shapes (BG1/BG2 at
small Z), 1024 codewords, one launch: ms per batch."""
import sys, json
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tools"))
import numpy as np
import paper_2009_05534_b200 as nr
from bench_configs import gpu_blocks, time_plan
res = {}
for bgn, z, ebn0 in ((2, 128, 1.0), (2, 192, 1.0), (1, 128, 2.0), (1, 64, 2.0)):
    bg = nr.load_basegraph(bgn, z)
    _, blocks = gpu_blocks(bg, bg.m_bg, ebn0, 1024, 3)
    plan = nr.Plan(bg, bg.m_bg, nr.DecodeConfig(max_iter=20, early_stop="syndrome"))
    out = plan.alloc_outputs(1024)
    res[f"bg{bgn}_z{z}"] = round(float(np.median(time_plan(plan, blocks, out, 20))), 4)
print(json.dumps(res))
