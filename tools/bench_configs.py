#!/usr/bin/env python
"""BASELINE.json configs 1, 3, 4 and 5 (config 2 is bench.py's headline).

Used by bench.py (its ``configs`` key) and runnable alone (one JSON line per
config). Device-resident timing with CUDA events on the launching streams;
inputs come from the reference's synthetic chain (encode, BPSK, AWGN,
L = 2y/sigma^2, quantize on the GPU).

  1  BG2 Z=64, one codeword, 10 fixed iterations: latency (harness.py:268-321
     protocol: warm-up, then per-rep timing, median and p99)
  3  BG2 Z=384, B=1024, Eb/N0 0.5 dB, syndrome early stop, max 20
     (decoder.py:497-523 semantics; the roofline counts the actual
     per-codeword iterations)
  4  all 51 Z x {BG1, BG2}, 16 codewords each (1632), 10 fixed iterations,
     one mixed batch (MixedBatchDecoder: one CUDA-graph replay)
  5  slot-scale: BG1 rows_used=8 (R~0.79), 7,488 codewords per launch
     (64 cell-slots x 117), Z in {384, 352, 320}; sharded across the given
     devices (strong scaling); latency against the 500 us slot

Each function returns (line, samples): ``samples`` is a list of
(bg, cfg, host int8 blocks, gpu outputs) for the caller's CPU-baseline /
parity leg. Nothing here touches oracle/.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import paper_2009_05534_b200 as nr  # noqa: E402
from paper_2009_05534_b200.shard import shard_bounds  # noqa: E402
from paper_2009_05534_b200.synth import noisy_llrs  # noqa: E402

OPS_PER_EDGE = 19


def edges_of(bg, rows):
    return int(bg.w_r[:rows].sum())


def gpu_blocks(bg, rows, ebn0, count, seed, device=0):
    params = nr.code_params(bg, bg.z, rows)
    msgs, llr = noisy_llrs(bg, rows, ebn0, count, seed)
    with torch.cuda.device(device):
        blocks = nr.quantize(torch.from_numpy(llr).to(f"cuda:{device}"), nr.QuantConfig(), params)
    return msgs, blocks


def host_sample(out, n):
    return {k: out[k][:n].cpu().numpy() for k in ("bits", "iters", "synd", "success")}


def roofline(ops, seconds, peak_ops):
    ach = ops / seconds
    return {"bound": "alu", "achieved": ach / 1e12, "peak": peak_ops / 1e12, "unit": "Tops/s",
            "frac": ach / peak_ops}


def time_plan(plan, blocks, out, reps, warm=5):
    for _ in range(warm):
        plan.decode_device(blocks, out)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        plan.decode_device(blocks, out)
        b.record()
    torch.cuda.synchronize()
    return np.array([a.elapsed_time(b) for a, b in ev])


def overlapped_ms(plan, blocks, batch, reps=40, nstreams=2):
    """Mean time per batch when independent batches alternate over streams."""
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    outs = [plan.alloc_outputs(batch) for _ in range(nstreams)]
    cur = torch.cuda.current_stream()

    def run(n):
        for s in streams:
            s.wait_stream(cur)
        for i in range(n):
            plan.decode_device(blocks, outs[i % nstreams], stream=streams[i % nstreams].cuda_stream)
        for s in streams:
            cur.wait_stream(s)

    run(2 * nstreams)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run(reps)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def config1(peak_ops, sms=148):
    bg = nr.load_basegraph("BG2", 64)
    cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
    plan = nr.get_plan(bg, 42, cfg)
    _, blocks = gpu_blocks(bg, 42, 4.0, 1, (0, 0))
    out = plan.alloc_outputs(1)
    t = time_plan(plan, blocks, out, 200)
    ops = OPS_PER_EDGE * edges_of(bg, 42) * 64 * 10
    p50 = float(np.median(t))
    rf = roofline(ops, p50 * 1e-3, peak_ops)
    rf["frac_one_sm"] = rf["frac"] * sms  # one codeword occupies one CTA on one SM
    line = {"config": 1, "workload": "BG2 Z=64 K=640, 1 codeword, 10 fixed iterations (latency)",
            "value": plan.k / (p50 * 1e-3) / 1e9, "unit": "Gbps",
            "p50_latency_us": p50 * 1e3, "p99_latency_us": float(np.percentile(t, 99) * 1e3),
            "per_iteration_us": p50 * 1e2, "reps": len(t), "roofline": rf,
            "roofline_note": "one codeword is one CTA of 2 warps on one SM: frac is against the whole "
                             "GPU, frac_one_sm against that SM's share of the peak"}
    return line, [(bg, cfg, blocks.cpu().numpy(), host_sample(out, 1))]


def config3(peak_ops):
    bg = nr.load_basegraph("BG2", 384)
    cfg = nr.DecodeConfig(max_iter=20)
    plan = nr.get_plan(bg, 42, cfg)
    msgs, blocks = gpu_blocks(bg, 42, 0.5, 1024, 3)
    out = plan.alloc_outputs(1024)
    t = time_plan(plan, blocks, out, 50)
    iters = out["iters"].cpu().numpy()
    bits = nr.unpack_bits(out["bits"].cpu().numpy(), plan.k)
    ovl = overlapped_ms(plan, blocks, 1024)
    ops = OPS_PER_EDGE * edges_of(bg, 42) * 384 * int(iters.sum())
    p50 = float(np.median(t))
    line = {"config": 3, "workload": "BG2 Z=384 K=3840, B=1024, Eb/N0 0.5 dB, syndrome stop, max 20",
            "value": 1024 * plan.k / (ovl * 1e-3) / 1e9, "unit": "Gbps",
            "value_note": "independent batches alternate over 2 streams (as the headline value)",
            "single_batch_value": 1024 * plan.k / (p50 * 1e-3) / 1e9,
            "p50_batch_ms": p50, "p99_batch_ms": float(np.percentile(t, 99)),
            "mean_iterations": float(iters.mean()), "iterations_min_max": [int(iters.min()), int(iters.max())],
            "bler": float((bits != msgs).any(axis=1).mean()),
            "roofline": roofline(ops, ovl * 1e-3, peak_ops),
            "roofline_note": "19 ops x 197 edges x Z x (sum of actual iterations) / overlapped batch time"}
    return line, [(bg, cfg, blocks[:64].cpu().numpy(), host_sample(out, 64))]


def config4(peak_ops, reps=30):
    """One mixed batch: 102 (graph, Z) groups of 16 codewords in one decode
    call (MixedBatchDecoder)."""
    from paper_2009_05534_b200.mixed import Group, MixedBatchDecoder
    cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
    groups, data = [], []
    for bg_id in ("BG1", "BG2"):
        for z in nr.ALL_LIFTING_SIZES:
            bg = nr.load_basegraph(bg_id, z)
            groups.append(Group(bg, bg.m_bg, 16))
            data.append(gpu_blocks(bg, bg.m_bg, 2.0, 16, (int(bg_id[-1]), z))[1])
    mixed = MixedBatchDecoder(groups, cfg, streams=24)
    for x, d in zip(mixed.inputs, data):
        x.copy_(d)
    mixed.capture()
    for _ in range(3):
        mixed.replay()
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        mixed.replay()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    total_k = sum(16 * p.k for p in mixed.plans)
    ops = sum(OPS_PER_EDGE * edges_of(g.bg, g.rows_used) * g.bg.z * 10 * 16 for g in groups)
    p50 = float(np.median(times))
    line = {"config": 4, "workload": "51 Z x {BG1,BG2}, 16 codewords each (1632 cw), 10 fixed iterations, "
                                     "one mixed batch",
            "path": mixed.describe(),
            "value": total_k / (p50 * 1e-3) / 1e9, "unit": "Gbps",
            "p50_batch_ms": p50, "p99_batch_ms": float(np.percentile(times, 99)),
            "roofline": roofline(ops, p50 * 1e-3, peak_ops)}
    samples = [(g.bg, cfg, x[:2].cpu().numpy(), host_sample(o, 2))
               for g, x, o in zip(groups, mixed.inputs, mixed.outputs)]
    return line, samples


def config5(peak_ops, devices=(0,), reps=15):
    """7,488 codewords (a third each at Z = 384, 352, 320), BG1 rows_used=8,
    split over ``devices`` (contiguous shards of every Z group, no
    collective); time = max over devices."""
    cfg = nr.DecodeConfig(max_iter=10, early_stop="none")
    per = 7488 // 3
    n = len(devices)
    jobs = []  # (device, bg, plan, blocks, out, stream)
    for z in (384, 352, 320):
        bg = nr.load_basegraph("BG1", z)
        _, full = gpu_blocks(bg, 8, 3.0, per, (5, z), device=devices[0])
        for i, d in enumerate(devices):
            lo, hi = shard_bounds(per, n, i)
            if hi <= lo:
                continue
            with torch.cuda.device(d):
                plan = nr.get_plan(bg, 8, cfg, device=d)
                blocks = full[lo:hi].to(f"cuda:{d}")
                jobs.append((d, bg, plan, blocks, plan.alloc_outputs(hi - lo), torch.cuda.Stream(device=d)))
    ev = {d: [] for d in devices}
    for rep in range(reps + 3):
        marks = {}
        for d in devices:
            with torch.cuda.device(d):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                cur = torch.cuda.current_stream(d)
                a.record(cur)
                marks[d] = (a, b, cur)
        for d, bg, plan, blocks, out, s in jobs:
            s.wait_stream(marks[d][2])
            plan.decode_device(blocks, out, stream=s.cuda_stream)
        for d, bg, plan, blocks, out, s in jobs:
            marks[d][2].wait_stream(s)
        for d in devices:
            marks[d][1].record(marks[d][2])
        for d in devices:
            torch.cuda.synchronize(d)
        if rep >= 3:
            for d in devices:
                ev[d].append(marks[d][0].elapsed_time(marks[d][1]))
    times = np.max(np.array([ev[d] for d in devices]), axis=0)
    total_k = sum(per * 22 * z for z in (384, 352, 320))
    ops = sum(OPS_PER_EDGE * 103 * z * 10 * per for z in (384, 352, 320))
    p50 = float(np.median(times))
    line = {"config": 5, "workload": "slot-scale: BG1 rows_used=8 (R~0.79), 7488 cw per launch "
                                     "(64 cell-slots x 117 cw), Z in {384,352,320} split 1/3 each",
            "devices": len(devices), "sharding": "contiguous shard of every Z group per device, no collective",
            "value": total_k / (p50 * 1e-3) / 1e9, "unit": "Gbps",
            "p50_latency_us": p50 * 1e3, "p99_latency_us": float(np.percentile(times, 99) * 1e3),
            "per_cell_slot_us": p50 * 1e3 / 64, "slot_budget_us": 500.0,
            "roofline": roofline(ops, p50 * 1e-3, peak_ops * len(devices))}
    samples = [(bg, cfg, blocks[:4].cpu().numpy(), host_sample(out, 4))
               for d, bg, plan, blocks, out, s in jobs if d == devices[0]]
    return line, samples


def run_all(peak_ops, devices=(0,), which=(1, 3, 4, 5)):
    lines, samples = [], []
    for c in which:
        t0 = time.time()
        if c == 5:
            line, smp = config5(peak_ops, devices)
        else:
            line, smp = {1: config1, 3: config3, 4: config4}[c](peak_ops)
        line["wall_s"] = round(time.time() - t0, 1)
        lines.append(line)
        samples.append(smp)
    return lines, samples


if __name__ == "__main__":
    import ctypes

    from paper_2009_05534_b200 import _native
    a, m = ctypes.c_double(), ctypes.c_double()
    _native.check(_native.load().nrldpc_alu_peak(0, ctypes.byref(a), ctypes.byref(m)))
    which = [int(x) for x in sys.argv[1:]] or [1, 3, 4, 5]
    lines, _ = run_all(2 * m.value, which=which)
    for line in lines:
        print(json.dumps(line), flush=True)
