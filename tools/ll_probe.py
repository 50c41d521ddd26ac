#!/usr/bin/env python
"""Single-codeword latency per iteration, the paper's Table 1 setting
(BG1 R=1/3 and BG2 R=1/5, LL-INT / LL-FP).

    python tools/ll_probe.py [reps]

Device-resident int8 blocks, 10 fixed iterations, CUDA events around each
launch (so one launch overhead is inside each sample); latency per iteration =
p50 / 10. Each case is parity-checked against the oracle.
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_05534_b200 as nr  # noqa: E402
from bench_configs import spot_check, time_plan  # noqa: E402
from paper_2009_05534_b200.synth import noisy_llrs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
cases = [("BG1", 384, 46, "BG1 R=1/3"), ("BG2", 384, 42, "BG2 R=1/5"), ("BG2", 64, 42, "BG2 Z=64 R=1/5"),
         ("BG1", 128, 46, "BG1 Z=128"), ("BG2", 192, 42, "BG2 Z=192"), ("BG1", 16, 46, "BG1 Z=16")]
out_lines = []
for name, z, rows, label in cases:
    bg = nr.load_basegraph(name, z)
    for prec in ("int8", "f16"):
        for batch in (1, 2):
            cfg = nr.DecodeConfig(max_iter=10, early_stop="none", precision=prec)
            plan = nr.Plan(bg, rows, cfg)
            params = nr.code_params(bg, z, rows)
            _, llr = noisy_llrs(bg, rows, 2.0, batch, seed=7)
            blocks = nr.quantize(torch.from_numpy(llr).cuda(), nr.QuantConfig(mode=prec), params)
            out = plan.alloc_outputs(batch)
            t = time_plan(plan, blocks, out, reps)
            ok = spot_check(plan, blocks, out, bg, cfg, n=batch)
            p50 = float(np.median(t)) * 1e3
            out_lines.append({"case": label, "z": z, "precision": prec, "batch": batch,
                              "p50_us": round(p50, 1), "per_iteration_us": round(p50 / 10, 2),
                              "p99_us": round(float(np.percentile(t, 99)) * 1e3, 1), "parity": ok})
            print(json.dumps(out_lines[-1]), flush=True)
