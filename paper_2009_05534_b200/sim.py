"""GPU link simulation: encode -> BPSK/AWGN/demap/quantize -> decode -> count.

The reference runs this loop on CPU processes (harness.run_bler_sweep,
/root/reference/pkg/src/ldpclab/harness.py:131-224; _run_batch :85-128).
Here every stage runs on the device:

* ``encode`` is the systematic encoder (``nrldpc_encode``), bit-exact with
  codec.encode_batch;
* ``channel`` is the fused BPSK + AWGN + L=2y/sigma^2 + int8 quantizer
  (``nrldpc_channel_awgn``, Philox normals). It is statistically, not
  draw-for-draw, equivalent to the reference's numpy stream;
* ``bler_sweep`` has the reference's stopping rule (target block errors or
  max codewords per Eb/N0 point) and returns the same SweepPoint fields.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .basegraph import code_params
from .channel import ebn0_to_sigma
from .decoder import DecodeConfig, EarlyStop, Precision, get_plan


def _stream(dev):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def encode(msgs, plan):
    """(B, K) uint8 0/1 CUDA tensor -> (B, n_c) uint8 codewords."""
    import torch
    msgs = msgs.to(torch.uint8).contiguous()
    out = torch.empty((msgs.shape[0], plan.n_c), dtype=torch.uint8, device=msgs.device)
    _native.check(_native.load().nrldpc_encode(plan.handle, msgs.data_ptr(), int(msgs.shape[0]),
                                               out.data_ptr(), _stream(msgs.device)))
    return out


def channel(codewords, plan, sigma: float, scale: float = 8.0, seed: int = 0):
    """(B, n_c) codeword bits -> (B, n_c) int8 decoder-domain LLR blocks."""
    import torch
    out = torch.empty(codewords.shape, dtype=torch.int8, device=codewords.device)
    _native.check(_native.load().nrldpc_channel_awgn(
        plan.handle, codewords.data_ptr(), int(codewords.shape[0]), float(sigma), float(scale),
        int(seed) & 0xFFFFFFFFFFFFFFFF, out.data_ptr(), _stream(codewords.device)))
    return out


def wilson_interval(k: int, n: int, z: float = 1.96) -> tuple[float, float]:
    if n == 0:
        return 0.0, 1.0
    p = k / n
    denom = 1.0 + z * z / n
    center = (p + z * z / (2 * n)) / denom
    half = z * math.sqrt(p * (1.0 - p) / n + z * z / (4 * n * n)) / denom
    return max(0.0, center - half), min(1.0, center + half)


@dataclass
class SweepPoint:
    ebn0_db: float
    sigma: float
    codewords: int
    bit_errors: int
    block_errors: int
    mean_iters: float
    median_iters: float
    wall_time_per_cw: float
    throughput_cbps: float
    info_bits: int = 0
    iterations: list = field(default_factory=list, repr=False)

    @property
    def bler(self) -> float:
        return self.block_errors / self.codewords if self.codewords else 0.0

    @property
    def ber(self) -> float:
        return self.bit_errors / (self.codewords * self.info_bits) if self.codewords else 0.0

    def wilson(self, z: float = 1.96):
        return wilson_interval(self.block_errors, self.codewords, z)


def bler_sweep(bg, rows_used: int, cfg: DecodeConfig, ebn0_grid, target_block_errors: int = 100,
               max_codewords: int = 100_000, seed: int = 0, scale: float = 8.0, batch: int = 4096,
               device: int = 0) -> list[SweepPoint]:
    """BLER/BER over an Eb/N0 grid, every stage on the GPU (int8 path)."""
    import torch
    if cfg.precision is not Precision.INT8:
        raise ValueError("the GPU channel model produces int8 blocks; use precision int8")
    if cfg.early_stop is EarlyStop.CRC:
        raise ValueError("bler_sweep draws raw messages; CRC payloads are not attached")
    if target_block_errors <= 0 or max_codewords <= 0:
        raise ValueError("stopping rule must be positive")
    params = code_params(bg, bg.z, rows_used)
    plan = get_plan(bg, rows_used, cfg, device)
    dev = torch.device("cuda", device)
    gen = torch.Generator(device=dev)
    points = []
    for p_idx, ebn0 in enumerate(ebn0_grid):
        sigma = ebn0_to_sigma(ebn0, params.k / params.n_tx) if not math.isinf(ebn0) else 1e-3
        gen.manual_seed(hash((seed, p_idx)) & 0x7FFFFFFFFFFFFFFF)
        total = blk = bit = 0
        iters_all = []
        t_dec = 0.0
        b_idx = 0
        while total < max_codewords and blk < target_block_errors:
            n = min(batch, max_codewords - total)
            msgs = torch.randint(0, 2, (n, params.k), dtype=torch.uint8, device=dev, generator=gen)
            blocks = channel(encode(msgs, plan), plan, sigma, scale, seed=(seed << 20) ^ (p_idx << 12) ^ b_idx)
            out = plan.alloc_outputs(n)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            plan.decode_device(blocks, out)
            torch.cuda.synchronize(dev)
            t_dec += time.perf_counter() - t0
            words = out["bits"].view(torch.int32)
            ref = torch.from_numpy(np.packbits(msgs.cpu().numpy(), axis=1, bitorder="little").view(np.uint8))
            got = torch.from_numpy(np.ascontiguousarray(words.cpu().numpy()).view(np.uint8)[:, : ref.shape[1]])
            diff = np.unpackbits((got ^ ref).numpy(), axis=1, bitorder="little")[:, : params.k]
            bit += int(diff.sum())
            blk += int(diff.any(axis=1).sum())
            iters_all.extend(out["iters"].cpu().numpy().tolist())
            total += n
            b_idx += 1
        points.append(SweepPoint(
            ebn0_db=ebn0, sigma=sigma, codewords=total, bit_errors=bit, block_errors=blk,
            mean_iters=float(np.mean(iters_all)), median_iters=float(np.median(iters_all)),
            wall_time_per_cw=t_dec / total, throughput_cbps=params.n_c * total / t_dec if t_dec else 0.0,
            info_bits=params.k, iterations=iters_all))
    return points
