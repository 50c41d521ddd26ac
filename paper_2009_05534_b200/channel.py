"""Channel side of the decode path.

``quantize`` is the GPU drop-in for ldpclab.channel.quantize
(/root/reference/pkg/src/ldpclab/channel.py:64-83): depuncture (2Z leading
zeros) and map channel LLRs into the decoder domain, computed in float64 on
the device exactly as the reference does on the host.

``bpsk_awgn`` / ``demap_llr`` / ``ebn0_to_sigma`` are host-side synthetic
traffic generators with the reference's semantics (channel.py:47-61, 86-95);
they drive the bench and BLER runs and are not part of the accelerated path.
"""

from __future__ import annotations

import ctypes
import math
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _native

INT8_MAX = 127
F16_MAX = 65504.0


@dataclass(frozen=True)
class QuantConfig:
    mode: str = "int8"
    scale: float = 8.0
    clip: float = math.inf

    def __post_init__(self):
        if self.mode not in ("int8", "f16", "f32"):
            raise ValueError(f"unknown quantization mode {self.mode!r}")
        if self.scale <= 0:
            raise ValueError("scale must be positive")


_MODE = {"int8": _native.INT8, "f16": _native.F16, "f32": _native.F32}


def bpsk_exact(bits) -> np.ndarray:
    return 1.0 - 2.0 * np.asarray(bits, dtype=np.float64)


def bpsk_awgn(bits, sigma: float, rng) -> np.ndarray:
    if sigma <= 0:
        raise ValueError("sigma must be positive (use bpsk_exact for the noise-disabled limit)")
    rng = np.random.default_rng(rng)
    sym = bpsk_exact(bits)
    return sym + rng.normal(0.0, sigma, size=sym.shape)


def demap_llr(symbols, sigma: float) -> np.ndarray:
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    return 2.0 * np.asarray(symbols, dtype=np.float64) / (sigma * sigma)


def ebn0_to_sigma(ebn0_db: float, rate_eff: float) -> float:
    if rate_eff <= 0:
        raise ValueError("effective rate must be positive")
    ebn0 = 10.0 ** (ebn0_db / 10.0)
    return math.sqrt(1.0 / (2.0 * rate_eff * ebn0))


_QPLANS: "OrderedDict" = OrderedDict()


def _quant_plan(params):
    # the quantize kernel only needs (Z, n_c); reuse one plan per shape (the
    # lookup is on the per-call path, so it must not rebuild graph tables)
    import torch
    key = (params.n_c, params.z, params.rows_used, torch.cuda.current_device())
    plan = _QPLANS.get(key)
    if plan is None:
        from .basegraph import load_basegraph
        from .decoder import PLAN_CACHE_MAX, DecodeConfig, get_plan
        k_b = params.n_c // params.z - params.rows_used
        bg = load_basegraph(1 if k_b == 22 else 2, params.z)
        plan = _QPLANS[key] = get_plan(bg, params.rows_used, DecodeConfig(), device=key[3])
        # bounded like the decoder's plan cache (least recently used out)
        while len(_QPLANS) > max(1, PLAN_CACHE_MAX):
            _QPLANS.popitem(last=False)
    else:
        _QPLANS.move_to_end(key)
    return plan


def quantize(llrs, cfg: QuantConfig, params):
    """Depuncture + quantize on the GPU. numpy in -> numpy out; a CUDA tensor
    in -> CUDA tensor out (asynchronous on the current stream)."""
    return _quantize(llrs, cfg, params, None)


def demap_quantize(symbols, sigma: float, cfg: QuantConfig, params):
    """Fused soft demapper + quantize (channel.py:57-61 then 64-83) on the
    GPU: received BPSK symbols in, decoder-domain LLR blocks out."""
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    return _quantize(symbols, cfg, params, float(sigma))


def _quantize(llrs, cfg, params, sigma):
    import torch
    out_dtype = {"int8": torch.int8, "f16": torch.float16, "f32": torch.float32}[cfg.mode]
    is_dev = type(llrs).__module__.split(".")[0] == "torch" and llrs.is_cuda
    if is_dev:
        x = llrs
        if x.dtype not in (torch.float64, torch.float32):
            x = x.to(torch.float64)
    else:
        x = torch.from_numpy(np.ascontiguousarray(np.asarray(llrs, dtype=np.float64)))
    if x.shape[-1] != params.n_tx:
        raise ValueError(f"expected {params.n_tx} LLRs, got {x.shape[-1]}")
    lead = tuple(x.shape[:-1])
    plan = _quant_plan(params)
    if not is_dev:
        x = x.to(f"cuda:{plan.device}")
    x = x.contiguous().reshape(-1, params.n_tx)
    out = torch.empty((x.shape[0], params.n_c), dtype=out_dtype, device=x.device)
    in_code = _native.IN_F64 if x.dtype == torch.float64 else _native.IN_F32
    stream = torch.cuda.current_stream(x.device).cuda_stream
    lib = _native.load()
    if sigma is None:
        _native.check(lib.nrldpc_quantize(
            plan.handle, x.data_ptr(), in_code, int(x.shape[0]), float(cfg.scale), float(cfg.clip),
            out.data_ptr(), _MODE[cfg.mode], ctypes.c_void_p(stream)))
    else:
        _native.check(lib.nrldpc_demap_quantize(
            plan.handle, x.data_ptr(), in_code, int(x.shape[0]), sigma, float(cfg.scale),
            float(cfg.clip), out.data_ptr(), _MODE[cfg.mode], ctypes.c_void_p(stream)))
    out = out.reshape(lead + (params.n_c,))
    return out if is_dev else out.cpu().numpy()
