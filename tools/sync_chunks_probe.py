#!/usr/bin/env python
"""Synchronous host-buffer decode (nrldpc_decode_host) wall time per call vs
the chunk count, BG1 Z=384, 1024 codewords from pinned int8: Gbps."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2009_05534_b200 as nr  # noqa: E402
from paper_2009_05534_b200.synth import noisy_llrs  # noqa: E402

bg = nr.load_basegraph(1, 384)
params = nr.code_params(bg, 384, 46)
plan = nr.get_plan(bg, 46, nr.DecodeConfig(max_iter=10, early_stop="none"))
B = 1024
_, llr = noisy_llrs(bg, 46, 2.0, 64, seed=1)
blk = nr.quantize(torch.from_numpy(llr).cuda(), nr.QuantConfig(), params).repeat(B // 64, 1)
host = torch.empty(blk.shape, dtype=torch.int8, pin_memory=True)
host.copy_(blk.cpu())
hin = host.numpy()
out = plan.host_outputs(B, pinned=True)
res = {}
for chunks in (4, 6, 8, 12, 16, 24, 32):
    for _ in range(3):
        plan.decode_host(hin, chunks=chunks, out=out)
    t0 = time.perf_counter()
    n = 30
    for _ in range(n):
        plan.decode_host(hin, chunks=chunks, out=out)
    dt = (time.perf_counter() - t0) / n
    res[chunks] = round(B * params.k / dt / 1e9, 2)
print(json.dumps(res))
