#!/usr/bin/env python
"""f16 / f32 engines with the syndrome stop (max 20) on BG1 Z=384 and BG2
Z=384, 1024 codewords, one launch: ms per batch and mean iterations."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_05534_b200 as nr  # noqa: E402
from bench_configs import time_plan  # noqa: E402
from paper_2009_05534_b200.synth import noisy_llrs  # noqa: E402

res = {}
for bgn, ebn0 in ((1, 2.0), (2, 0.5)):
    bg = nr.load_basegraph(bgn, 384)
    params = nr.code_params(bg, 384, bg.m_bg)
    _, llr = noisy_llrs(bg, bg.m_bg, ebn0, 256, seed=5)
    for prec in ("f16", "f32"):
        q = nr.quantize(torch.from_numpy(llr).cuda(), nr.QuantConfig(mode=prec), params).repeat(4, 1)
        plan = nr.Plan(bg, bg.m_bg, nr.DecodeConfig(max_iter=20, early_stop="syndrome", precision=prec))
        out = plan.alloc_outputs(1024)
        t = float(np.median(time_plan(plan, q, out, 10)))
        res[f"bg{bgn}_{prec}"] = {"ms": round(t, 4), "mean_it": round(float(out["iters"].float().mean()), 2)}
print(json.dumps(res))
