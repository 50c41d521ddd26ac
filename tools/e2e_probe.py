"""Host->device pipeline probe: H2D chunks on one copy stream, chunk decodes
on compute streams, one D2H at the end; device-timed with events."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2009_05534_b200 as nr  # noqa: E402
from paper_2009_05534_b200.synth import noisy_llrs  # noqa: E402

bg = nr.load_basegraph(1, 384)
params = nr.code_params(bg, 384, 46)
cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
plan = nr.get_plan(bg, 46, cfg)
B = 1024
_, llr = noisy_llrs(bg, 46, 2.0, 64, seed=1)
blk = nr.quantize(torch.from_numpy(llr).cuda(), nr.QuantConfig(), params)
blk = blk.repeat(B // 64, 1)
h = torch.empty(blk.shape, dtype=torch.int8, pin_memory=True)
h.copy_(blk.cpu())
d = torch.empty_like(blk)
out = plan.alloc_outputs(B)
hb = torch.empty(out["bits"].shape, dtype=out["bits"].dtype, pin_memory=True)
cp = torch.cuda.Stream()
comp = [torch.cuda.Stream() for _ in range(8)]


def run(chunks, ncomp, first_frac=None):
    sizes = [B // chunks] * chunks
    evs = []
    b0 = 0
    for i, n in enumerate(sizes):
        with torch.cuda.stream(cp):
            d[b0:b0 + n].copy_(h[b0:b0 + n], non_blocking=True)
            e = torch.cuda.Event()
            e.record(cp)
        s = comp[i % ncomp]
        s.wait_event(e)
        o = {k: v[b0:b0 + n] for k, v in out.items()}
        plan.decode_device(d[b0:b0 + n], o, stream=s.cuda_stream)
        b0 += n
    for s in comp[:ncomp]:
        cp.wait_stream(s)
    with torch.cuda.stream(cp):
        hb.copy_(out["bits"], non_blocking=True)


for chunks, ncomp in ((1, 1), (2, 2), (4, 4), (8, 4), (8, 8), (16, 8), (32, 8)):
    for _ in range(3):
        run(chunks, ncomp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(20):
        e0.record(cp)
        for s in comp:
            s.wait_stream(cp)
        run(chunks, ncomp)
        e1.record(cp)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    print(f"chunks={chunks:2d} comp_streams={ncomp}: {ms:.3f} ms  {B * params.k / ms / 1e6:.2f} Gbps")

# sequential breakdown on one stream
s = torch.cuda.current_stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for rep in range(3):
    torch.cuda.synchronize()
    ev[0].record(s)
    d.copy_(h, non_blocking=True)
    ev[1].record(s)
    plan.decode_device(d, out, stream=s.cuda_stream)
    ev[2].record(s)
    hb.copy_(out["bits"], non_blocking=True)
    ev[3].record(s)
    torch.cuda.synchronize()
print("H2D %.3f  decode %.3f  D2H %.3f ms" % tuple(ev[i].elapsed_time(ev[i + 1]) for i in range(3)))
# decode of an L2-cold vs just-copied input
torch.cuda.synchronize()
ev[0].record(s)
plan.decode_device(d, out, stream=s.cuda_stream)
ev[1].record(s)
torch.cuda.synchronize()
print("decode alone %.3f ms" % ev[0].elapsed_time(ev[1]))
