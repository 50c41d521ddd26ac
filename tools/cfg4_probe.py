"""Config 4 (mixed batch, 102 groups x 16 codewords): where the time goes.
Replay time vs the number of side streams, and for subsets of the groups
(only the shapes that hold an SM alone, only the rest)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2009_05534_b200 as nr  # noqa: E402
from paper_2009_05534_b200.mixed import Group, MixedBatchDecoder  # noqa: E402


def replay_ms(mixed, reps=20):
    mixed.capture()
    for _ in range(3):
        mixed.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        mixed.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
groups = []
for bg_id in ("BG1", "BG2"):
    for z in nr.ALL_LIFTING_SIZES:
        bg = nr.load_basegraph(bg_id, z)
        groups.append(Group(bg, bg.m_bg, 16))
k_total = sum(16 * g.bg.k_b * g.bg.z for g in groups)
for grouped in (True, False):
    for streams in (8, 16, 32, 64):
        m = MixedBatchDecoder(groups, cfg, streams=streams, grouped=grouped)
        t = replay_ms(m)
        print(f"grouped={grouped} launches={len(m.launches)} streams={streams:3d}: {t:.3f} ms  "
              f"{k_total / t / 1e6:.2f} Gbps")
m = MixedBatchDecoder(groups, cfg, streams=32, grouped=False)
alone = [g for g, p in zip(groups, m.plans) if p.smem_bytes > 116 * 1024 or p.threads_per_cta >= 384]
rest = [g for g, p in zip(groups, m.plans) if not (p.smem_bytes > 116 * 1024 or p.threads_per_cta >= 384)]
print("groups holding an SM alone:", len(alone), "ms", replay_ms(MixedBatchDecoder(alone, cfg, streams=32, grouped=False)))
print("other groups:", len(rest), "ms", replay_ms(MixedBatchDecoder(rest, cfg, streams=32, grouped=False)))
print("groups holding an SM alone, grouped:", replay_ms(MixedBatchDecoder(alone, cfg, streams=32)))
print("other groups, grouped:", replay_ms(MixedBatchDecoder(rest, cfg, streams=32)))
for g, p in zip(groups, m.plans):
    print(f"  {g.bg.id} Z={g.bg.z:3d} threads={p.threads_per_cta:3d} cw/cta={p.codewords_per_cta} smem={p.smem_bytes}")


print("-- grouped, stream count and launch order")
class ShortFirst(MixedBatchDecoder):
    def _schedule(self, n):
        return list(reversed(super()._schedule(n)))
for st in (20, 24, 28, 32, 33, 40, 48):
    print(f"grouped LPT streams={st}: {replay_ms(MixedBatchDecoder(groups, cfg, streams=st)):.3f} ms   "
          f"short-first: {replay_ms(ShortFirst(groups, cfg, streams=st)):.3f} ms")

print("-- plans without the co-scheduling hint (ABS / TM variants where they apply)")
for st in (16, 24, 32):
    print(f"grouped, coscheduled=False, streams={st}: "
          f"{replay_ms(MixedBatchDecoder(groups, cfg, streams=st, coscheduled=False)):.3f} ms")
