"""Per-CTA fixed cost of the headline kernel: one full wave (148 pair-CTAs,
296 codewords, BG1 Z=384) timed at several fixed iteration counts; the
intercept of time vs iterations is the prologue + final check + result
writes, the slope one iteration."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import paper_2009_05534_b200 as nr  # noqa: E402
from bench_configs import gpu_blocks, time_plan  # noqa: E402

bg = nr.load_basegraph("BG1", 384)
sms = torch.cuda.get_device_properties(0).multi_processor_count
B = 2 * sms
_, blocks = gpu_blocks(bg, 46, 2.0, B, (2024, 0))
xs, ys = [], []
for it in (1, 2, 5, 10, 20):
    plan = nr.Plan(bg, 46, nr.DecodeConfig(max_iter=it, early_stop="none"))
    out = plan.alloc_outputs(B)
    t = float(np.median(time_plan(plan, blocks, out, 50))) * 1e3
    xs.append(it)
    ys.append(t)
    print(f"iterations {it:2d}: {t:8.2f} us per wave ({B} codewords)")
slope, icpt = np.polyfit(xs, ys, 1)
print(f"fit: {slope:.2f} us per iteration, {icpt:.2f} us fixed per CTA (prologue + final check + writes + launch)")
