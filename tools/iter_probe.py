#!/usr/bin/env python
"""Single-launch time vs fixed iteration count (BG1 Z=384): separates the
per-iteration cost from the per-CTA fixed cost (prologue, final check, bit
writes, CTA scheduling).

    python tools/iter_probe.py
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import numpy as np  # noqa: E402

import paper_2009_05534_b200 as nr  # noqa: E402
from bench_configs import gpu_blocks, time_plan  # noqa: E402

bg = nr.load_basegraph(1, 384)
_, blocks = gpu_blocks(bg, 46, 2.0, 1024, 1)
for batch in (296, 1024):
    res = {"batch": batch}
    for it in (1, 2, 5, 10, 20):
        plan = nr.Plan(bg, 46, nr.DecodeConfig(max_iter=it, early_stop="none"))
        out = plan.alloc_outputs(batch)
        res[it] = round(float(np.median(time_plan(plan, blocks[:batch], out, 20))) * 1e3, 1)
    print(json.dumps(res), flush=True)
