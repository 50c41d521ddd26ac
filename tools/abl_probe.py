#!/usr/bin/env python
"""Timing-only A/B of alternative builds of libnrldpc.so (ablation variants
give wrong results; only their timing is read).

    python tools/abl_probe.py lib1.so [lib2.so ...]   (one process per lib)
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

if len(sys.argv) > 1 and sys.argv[1] != "--one":
    for so in sys.argv[1:]:
        out = subprocess.run([sys.executable, __file__, "--one", so], capture_output=True, text=True)
        print(so, out.stdout.strip() or out.stderr[-2000:], flush=True)
    sys.exit(0)

os.environ["NRLDPC_LIB"] = sys.argv[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import numpy as np  # noqa: E402

import paper_2009_05534_b200 as nr  # noqa: E402
from bench_configs import gpu_blocks, overlapped_ms, time_plan  # noqa: E402

res = {}
for bgn, z in ((1, 384), (2, 384), (1, 256)):
    bg = nr.load_basegraph(bgn, z)
    plan = nr.Plan(bg, bg.m_bg, nr.DecodeConfig(max_iter=10, early_stop="none"))
    _, blocks = gpu_blocks(bg, bg.m_bg, 2.0, 1024, 1)
    out = plan.alloc_outputs(1024)
    t = time_plan(plan, blocks, out, 40)
    res[f"bg{bgn}_z{z}_ms"] = round(float(np.median(t)), 4)
    res[f"bg{bgn}_z{z}_ovl_ms"] = round(float(overlapped_ms(plan, blocks, 1024)), 4)
print(json.dumps(res))
