"""Throughput of the f16 / f32 / int8 engines on the headline shape."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import paper_2009_05534_b200 as nr  # noqa: E402
from bench_configs import time_plan  # noqa: E402
from paper_2009_05534_b200.synth import noisy_llrs  # noqa: E402

bg = nr.load_basegraph(1, 384)
params = nr.code_params(bg, 384, 46)
B = 1024
_, llr = noisy_llrs(bg, 46, 2.0, 64, seed=1)
for prec in ("int8", "f16", "f32"):
    cfg = nr.DecodeConfig(max_iter=10, early_stop="none", precision=prec)
    plan = nr.get_plan(bg, 46, cfg)
    q = nr.quantize(torch.from_numpy(llr).cuda(), nr.QuantConfig(mode=prec), params).repeat(B // 64, 1)
    out = plan.alloc_outputs(B)
    t = time_plan(plan, q, out, 10)
    ms = float(np.median(t))
    print(f"{prec}: {ms:.3f} ms per {B} codewords, {B * params.k / ms / 1e6:.2f} Gbps, "
          f"lanes={plan.lanes} threads/cta={plan.threads_per_cta} smem={plan.smem_bytes}")
