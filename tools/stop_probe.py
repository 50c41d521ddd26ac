#!/usr/bin/env python
"""Where the early-stop time goes (config 3 shape: BG2 Z=384, B=1024).

    python tools/stop_probe.py [bg] [z]

Prints the fixed-iteration cost per iteration (slope between 10 and 20
iterations), the syndrome-stop time at several SNRs next to the time the same
total iteration count would take at the fixed-iteration rate, and the all-fail
case (-3 dB: every codeword runs max_iter with the per-iteration check) next
to fixed 20 iterations.
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import numpy as np  # noqa: E402

import paper_2009_05534_b200 as nr  # noqa: E402
from bench_configs import gpu_blocks, time_plan  # noqa: E402

bgn = int(sys.argv[1]) if len(sys.argv) > 1 else 2
z = int(sys.argv[2]) if len(sys.argv) > 2 else 384
B = 1024
bg = nr.load_basegraph(bgn, z)
rows = bg.m_bg
_, blocks = gpu_blocks(bg, rows, 0.5, B, 7)
fixed = {}
for it in (10, 20):
    plan = nr.Plan(bg, rows, nr.DecodeConfig(max_iter=it, early_stop="none"))
    out = plan.alloc_outputs(B)
    fixed[it] = float(np.median(time_plan(plan, blocks, out, 20)))
slope = (fixed[20] - fixed[10]) / 10
base = fixed[10] - 10 * slope
print(json.dumps({"fixed_ms": fixed, "per_iteration_ms": round(slope, 4), "intercept_ms": round(base, 4)}))
for ebn0 in (-3.0, 0.5, 1.5, 3.0):
    _, bl = gpu_blocks(bg, rows, ebn0, B, 7)
    res = {"ebn0": ebn0}
    for flag in ("refill", "pairs"):
        if flag == "pairs":
            os.environ["NRLDPC_NO_REFILL"] = "1"
        else:
            os.environ.pop("NRLDPC_NO_REFILL", None)
        plan = nr.Plan(bg, rows, nr.DecodeConfig(max_iter=20, early_stop="syndrome"))
        out = plan.alloc_outputs(B)
        t = float(np.median(time_plan(plan, bl, out, 20)))
        its = out["iters"].cpu().numpy()
        # the fixed-iteration rate applied to the same work
        ideal = base + its.mean() * slope
        res[flag] = {"ms": round(t, 4), "mean_it": round(float(its.mean()), 2), "max_it": int(its.max()),
                     "fixed_rate_equiv_ms": round(ideal, 4), "overhead": round(t / ideal - 1, 3)}
    os.environ.pop("NRLDPC_NO_REFILL", None)
    print(json.dumps(res), flush=True)
