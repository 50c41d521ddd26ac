#!/usr/bin/env python
"""Single-launch and 1/2/3-stream overlapped batch time (ms per 1024-codeword
batch, 10 fixed iterations) for BG2 Z=384, BG1 Z=256 and BG1 Z=384; run with
and without NRLDPC_NO_TM=1 to compare the TM and byte-pair layouts.

    python tools/ovl_probe.py
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
from bench_configs import gpu_blocks, overlapped_ms, time_plan  # noqa: E402
res = {}
for bgn, z in ((2, 384), (1, 256), (1, 384)):
    bg = nr.load_basegraph(bgn, z)
    plan = nr.Plan(bg, bg.m_bg, nr.DecodeConfig(max_iter=10, early_stop="none"))
    _, blocks = gpu_blocks(bg, bg.m_bg, 2.0, 1024, 1)
    out = plan.alloc_outputs(1024)
    r = {"smem": plan.smem_bytes, "single": round(float(np.median(time_plan(plan, blocks, out, 30))), 4)}
    for ns in (1, 2, 3):
        r[f"ovl{ns}"] = [round(float(overlapped_ms(plan, blocks, 1024, nstreams=ns)), 4) for _ in range(2)]
    res[f"bg{bgn}_z{z}"] = r
print(os.environ.get("NRLDPC_NO_TM", "tm"), json.dumps(res))
