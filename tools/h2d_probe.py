import torch, time
n = 26738688
h = torch.empty(n, dtype=torch.int8, pin_memory=True)
d = torch.empty(n, dtype=torch.int8, device="cuda")
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
for chunks in (1, 4, 16):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        step = n // chunks
        for c in range(chunks):
            d[c*step:(c+1)*step].copy_(h[c*step:(c+1)*step], non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"H2D {n/1e6:.1f} MB in {chunks} pieces: {ms:.3f} ms  {n/ms/1e6:.1f} GB/s")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): h.copy_(d, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"D2H {ms:.3f} ms {n/ms/1e6:.1f} GB/s")
