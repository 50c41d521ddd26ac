"""Quantize kernel throughput vs HBM (f64 LLRs in, int8 out) for BG1 Z=384 B=1024."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2009_05534_b200 as nr  # noqa: E402

bg = nr.load_basegraph(1, 384)
params = nr.code_params(bg, 384, 46)
B = 1024
x = torch.randn(B, params.n_tx, dtype=torch.float64, device="cuda") * 3
for dt in (torch.float64, torch.float32):
    xi = x.to(dt)
    for _ in range(3):
        nr.quantize(xi, nr.QuantConfig(), params)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        nr.quantize(xi, nr.QuantConfig(), params)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    nbytes = B * params.n_tx * xi.element_size() + B * params.n_c
    print(f"{dt}: {ms * 1e3:.1f} us per call, {nbytes / ms / 1e6:.0f} GB/s")
