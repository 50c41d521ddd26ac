"""Syndrome-stop throughput with and without lane refill (plans created with
and without NRLDPC_NO_REFILL set, timed alternately)."""
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

for bgn, z, ebn0, mx in ((1, 384, 2.0, 20), (1, 384, 3.0, 20), (2, 384, 0.5, 20), (2, 384, 1.5, 20)):
    bg = nr.load_basegraph(bgn, z)
    cfg = nr.DecodeConfig(max_iter=mx, early_stop="syndrome")
    _, blocks = gpu_blocks(bg, bg.m_bg, ebn0, 1024, 7)
    plan = nr.Plan(bg, bg.m_bg, cfg)
    out = plan.alloc_outputs(1024)
    res = {}
    for flag in ("refill", "pairs"):
        if flag == "pairs":
            os.environ["NRLDPC_NO_REFILL"] = "1"
        else:
            os.environ.pop("NRLDPC_NO_REFILL", None)
        res[flag] = float(np.median(time_plan(plan, blocks, out, 20)))
    os.environ.pop("NRLDPC_NO_REFILL", None)
    it = out["iters"].float()
    k = plan.k
    print(f"BG{bgn} Z={z} {ebn0} dB: mean it {it.mean():.1f} (max {int(it.max())}); "
          f"pairs {res['pairs']:.3f} ms {1024 * k / res['pairs'] / 1e6:.2f} Gbps | "
          f"refill {res['refill']:.3f} ms {1024 * k / res['refill'] / 1e6:.2f} Gbps")
