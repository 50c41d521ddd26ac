"""BASELINE config 4 mixed batch (102 groups x 16 codewords), replayed a few
times; for ncu captures of the per-shape kernels (tools/profile_r02.sh)."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import bench_configs  # noqa: E402

if __name__ == "__main__":
    line, _ = bench_configs.config4(64e12, reps=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
    torch.cuda.synchronize()
    print(line["value"], line["p50_batch_ms"])
