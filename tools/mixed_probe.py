#!/usr/bin/env python
"""Mixed-batch probe: MixedBatchDecoder over a subset of (graph, Z) groups.

    python tools/mixed_probe.py [bgs=12] [zmin=2] [zmax=384] [count=16] [streams=32]
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import paper_2009_05534_b200 as nr  # noqa: E402
from paper_2009_05534_b200.mixed import Group, MixedBatchDecoder  # noqa: E402
from bench_configs import gpu_blocks  # noqa: E402

a = sys.argv[1:] + [None] * 5
bgs = a[0] or "12"
zmin, zmax = int(a[1] or 2), int(a[2] or 384)
count, streams = int(a[3] or 16), int(a[4] or 32)
cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
groups, data = [], []
zs = [int(v) for v in os.environ["PROBE_ZS"].split(",")] if os.environ.get("PROBE_ZS") else nr.ALL_LIFTING_SIZES
for b in bgs:
    for z in zs:
        if not zmin <= z <= zmax:
            continue
        if os.environ.get("PROBE_ZMOD") and z % int(os.environ["PROBE_ZMOD"]):
            continue
        bg = nr.load_basegraph(int(b), z)
        groups.append(Group(bg, bg.m_bg, count))
        data.append(gpu_blocks(bg, bg.m_bg, 2.0, count, (int(b), z))[1])
mixed = MixedBatchDecoder(groups, cfg, streams=streams)
for x, d in zip(mixed.inputs, data):
    x.copy_(d)
mixed.capture()
for _ in range(3):
    mixed.replay()
torch.cuda.synchronize()
ts = []
for _ in range(int(os.environ.get("PROBE_REPS", "15"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mixed.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"bgs={bgs} z=[{zmin},{zmax}] groups={len(groups)} count={count} streams={streams} "
      f"p50_ms={np.median(ts):.3f}")
