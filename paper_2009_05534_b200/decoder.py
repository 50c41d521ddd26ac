"""Drop-in layered min-sum decode on B200: ``decode(llrs, bg, cfg, trace=None)``.

Mirrors the reference's public decode surface
(/root/reference/pkg/src/ldpclab/decoder.py):

* ``Strategy`` / ``Precision`` / ``EarlyStop`` enums (decoder.py:32-46),
* ``DecodeConfig`` with the same fields, defaults and ``ValueError`` messages
  (decoder.py:49-85),
* ``DecodeResult`` (decoder.py:88-96),
* ``decode`` with the same input validation and result semantics
  (decoder.py:256-292, 486-566), including the ``trace`` list of
  ``(codeword, iteration, syndrome_weight, min|L_v|)``.

Every decode runs the sm_100a kernel in ``libnrldpc.so`` through the C ABI
(``_native``); there is no CPU path. ``bg`` may be this package's
``BaseGraph`` or the reference's ``ldpclab.BaseGraph`` (only ``id``, ``k_b``,
``m_bg``, ``z`` and ``row_entries`` are read).

``Strategy`` and ``alpha`` select how the reference *emulates* the paper's
thread shapes; results are bit-identical across strategies (decoder.py:10-14,
tests/test_acceptance.py:117-135) and across rho (decoder.py:3-8), so they are
validated and otherwise only affect the trace grouping for rho=4.
"""

from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _native
from .basegraph import edge_tables

INT8_SAT = 127


class Strategy(str, Enum):
    HIGH_THROUGHPUT = "high_throughput"
    LOW_LATENCY = "low_latency"


class Precision(str, Enum):
    INT8 = "int8"
    F16 = "f16"
    F32 = "f32"


class EarlyStop(str, Enum):
    SYNDROME = "syndrome"
    CRC = "crc"
    NONE = "none"


@dataclass(frozen=True)
class DecodeConfig:
    """Decoder knobs; validated exactly like the reference (decoder.py:62-85)."""

    beta: float = 0.75
    max_iter: int = 20
    strategy: Strategy = Strategy.HIGH_THROUGHPUT
    alpha: int = 4
    rho: int = 1
    precision: Precision = Precision.INT8
    early_stop: EarlyStop = EarlyStop.SYNDROME
    crc_kind: str = "crc24b"

    def __post_init__(self):
        if not 0.0 < self.beta <= 1.0:
            raise ValueError("beta must be in (0, 1]")
        if self.max_iter < 1:
            raise ValueError("max_iter must be at least 1")
        strategy = Strategy(_enum_value(self.strategy))
        precision = Precision(_enum_value(self.precision))
        early = EarlyStop(_enum_value(self.early_stop))
        object.__setattr__(self, "strategy", strategy)
        object.__setattr__(self, "precision", precision)
        object.__setattr__(self, "early_stop", early)
        if strategy is Strategy.LOW_LATENCY:
            if self.alpha < 1 or self.alpha & (self.alpha - 1):
                raise ValueError("alpha must be a power of two for low latency")
        allowed_rho = {Precision.INT8: (1, 4), Precision.F16: (1, 2), Precision.F32: (1,)}[precision]
        if self.rho not in allowed_rho:
            raise ValueError(
                f"rho={self.rho} is inconsistent with precision {precision.value} "
                f"(allowed: {allowed_rho})")


def _enum_value(x):
    # accept the reference's enums (same string values) as well as ours
    return x.value if isinstance(x, Enum) else x


@dataclass
class DecodeResult:
    bits: np.ndarray              # (B, K) uint8 hard decisions on information bits
    iterations: np.ndarray        # (B,) int64
    success: np.ndarray           # (B,) bool
    syndrome_weight: np.ndarray   # (B,) int64
    crc_ok: np.ndarray | None = None


_FLOAT_DTYPE = {Precision.F16: np.float16, Precision.F32: np.float32}
_PREC_CODE = {Precision.INT8: _native.INT8, Precision.F16: _native.F16, Precision.F32: _native.F32}
_STOP_CODE = {EarlyStop.SYNDROME: _native.STOP_SYNDROME, EarlyStop.CRC: _native.STOP_CRC,
              EarlyStop.NONE: _native.STOP_NONE}


class Plan:
    """Owns one ``nrldpc_plan`` (graph tables + config baked for one device)."""

    def __init__(self, bg, rows_used: int, cfg: DecodeConfig, device: int = 0, coscheduled: bool = False):
        lib = _native.load()
        self.tables = edge_tables(bg, rows_used)
        self.cfg = cfg
        self.device = device
        handle = ctypes.c_void_p()
        t = self.tables
        if cfg.crc_kind not in _native.CRC_KINDS:
            raise ValueError(f"unknown CRC kind {cfg.crc_kind!r}; choose from {sorted(_native.CRC_KINDS)}")
        _native.check(lib.nrldpc_plan_create(
            device, t.k_b, t.z, t.rows_used,
            t.row_start.ctypes.data, t.cols.ctypes.data, t.shifts.ctypes.data,
            _PREC_CODE[cfg.precision], float(cfg.beta), int(cfg.max_iter),
            _STOP_CODE[cfg.early_stop], _native.CRC_KINDS[cfg.crc_kind], ctypes.byref(handle)))
        self.handle = handle
        self.coscheduled = bool(coscheduled)
        if coscheduled:
            # launches share SMs with other plans' (mixed-shape batches)
            _native.check(lib.nrldpc_plan_set_coscheduled(handle, 1))
        vals = [ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(),
                ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()]
        _native.check(lib.nrldpc_plan_info(handle, *[ctypes.byref(v) for v in vals]))
        (self.k, self.n_c, self.n_tx, self.words, self.lanes, self.groups_per_cta,
         self.threads_per_cta, self.smem_bytes) = [v.value for v in vals]

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _native._lib is not None:
            _native._lib.nrldpc_plan_destroy(h)
            self.handle = None

    @property
    def codewords_per_cta(self) -> int:
        return self.groups_per_cta * self.lanes

    # -- device-resident path (torch CUDA tensors in and out) ---------------
    def alloc_outputs(self, batch: int, trace: bool = False):
        import torch
        dev = torch.device("cuda", self.device)
        out = {
            "bits": torch.empty((batch, self.words), dtype=torch.int32, device=dev),
            "iters": torch.empty(batch, dtype=torch.int32, device=dev),
            "synd": torch.empty(batch, dtype=torch.int32, device=dev),
            "success": torch.empty(batch, dtype=torch.uint8, device=dev),
            "crc_ok": torch.empty(batch, dtype=torch.uint8, device=dev),
            "status": torch.zeros(1, dtype=torch.int32, device=dev),
        }
        if trace:
            out["trace_w"] = torch.empty((batch, self.cfg.max_iter), dtype=torch.int32, device=dev)
            out["trace_m"] = torch.empty((batch, self.cfg.max_iter), dtype=torch.float32, device=dev)
        return out

    def decode_flooding_device(self, llr, out: dict, stream=None) -> None:
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        tw = out.get("trace_w")
        tm = out.get("trace_m")
        _native.check(_native.load().nrldpc_decode_flooding(
            self.handle, llr.data_ptr(), int(llr.shape[0]),
            out["bits"].data_ptr(), out["iters"].data_ptr(), out["synd"].data_ptr(),
            out["success"].data_ptr(), out["crc_ok"].data_ptr(),
            tw.data_ptr() if tw is not None else None, tm.data_ptr() if tm is not None else None,
            out["status"].data_ptr() if "status" in out else None,
            stream))

    def decode_device(self, llr, out: dict, stream=None) -> None:
        """Asynchronous decode of a CUDA tensor (B, n_c) into ``out`` buffers."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        batch = int(llr.shape[0])
        tw = out.get("trace_w")
        tm = out.get("trace_m")
        _native.check(_native.load().nrldpc_decode(
            self.handle, llr.data_ptr(), batch,
            out["bits"].data_ptr(), out["iters"].data_ptr(), out["synd"].data_ptr(),
            out["success"].data_ptr(),
            out["crc_ok"].data_ptr() if "crc_ok" in out else None,
            tw.data_ptr() if tw is not None else None,
            tm.data_ptr() if tm is not None else None,
            out["status"].data_ptr() if "status" in out else None,
            stream))

    # -- host-buffer path (the end-to-end C-ABI call) -----------------------
    def host_outputs(self, batch: int, pinned: bool = False) -> dict:
        shapes = {"bits": ((batch, self.words), np.uint32), "iters": ((batch,), np.int32),
                  "synd": ((batch,), np.int32), "success": ((batch,), np.uint8),
                  "crc_ok": ((batch,), np.uint8)}
        if not pinned:
            return {k: np.empty(s, d) for k, (s, d) in shapes.items()}
        import torch

        from .hostmem import pinned_empty
        tdt = {np.uint32: torch.int32, np.int32: torch.int32, np.uint8: torch.uint8}
        out = {}
        for k, (s, d) in shapes.items():
            out[k] = pinned_empty(s, tdt[d], self.device).numpy().view(d)  # on the GPU's NUMA node
        return out

    def decode_host_async(self, llr: np.ndarray, chunks: int = 12, out: dict | None = None) -> tuple[int, dict]:
        """Enqueue a host-buffer decode (nrldpc_decode_host_async); returns
        (ticket, out). ``llr`` and ``out`` must stay alive (and should be
        pinned) until ``host_wait(ticket)``."""
        batch = int(llr.shape[0])
        if not llr.flags.c_contiguous:
            raise ValueError("llr must be C-contiguous")
        if out is None:
            out = self.host_outputs(batch)
        t = ctypes.c_int64()
        _native.check(_native.load().nrldpc_decode_host_async(
            self.handle, llr.ctypes.data, batch, out["bits"].ctypes.data, out["iters"].ctypes.data,
            out["synd"].ctypes.data, out["success"].ctypes.data, out["crc_ok"].ctypes.data,
            int(chunks), ctypes.byref(t)))
        return t.value, out

    def host_wait(self, ticket: int) -> None:
        _native.check(_native.load().nrldpc_host_wait(self.handle, int(ticket)))

    def decode_host(self, llr: np.ndarray, chunks: int = 4, out: dict | None = None) -> dict:
        """Synchronous end-to-end decode of HOST buffers through the C ABI
        (H2D copy, kernel, D2H copy pipelined over ``chunks`` sub-batches)."""
        batch = int(llr.shape[0])
        llr = np.ascontiguousarray(llr)
        if out is None:
            out = self.host_outputs(batch)
        _native.check(_native.load().nrldpc_decode_host(
            self.handle, llr.ctypes.data, batch, out["bits"].ctypes.data, out["iters"].ctypes.data,
            out["synd"].ctypes.data, out["success"].ctypes.data, out["crc_ok"].ctypes.data,
            int(chunks)))
        return out

    def decode_host_bytes(self, llr: np.ndarray, chunks: int = 4) -> dict:
        """decode_host with the hard decisions as the reference's (B, K) bytes
        (nrldpc_decode_host_bytes): each chunk's words are unpacked by the
        library's host threads while later chunks still decode."""
        batch = int(llr.shape[0])
        llr = np.ascontiguousarray(llr)
        out = {"bits": np.empty((batch, self.k), np.uint8), "iters": np.empty(batch, np.int32),
               "synd": np.empty(batch, np.int32), "success": np.empty(batch, np.uint8),
               "crc_ok": np.empty(batch, np.uint8)}
        _native.check(_native.load().nrldpc_decode_host_bytes(
            self.handle, llr.ctypes.data, batch, out["bits"].ctypes.data, out["iters"].ctypes.data,
            out["synd"].ctypes.data, out["success"].ctypes.data, out["crc_ok"].ctypes.data, int(chunks)))
        return out


# Plans cached per (graph, Z, rows_used, config, device), least recently used
# first out. An evicted plan is destroyed (nrldpc_plan_destroy: its streams,
# events and staging buffers) once nothing else holds it, so a long BLER sweep
# over many shapes through the drop-in keeps a bounded footprint.
PLAN_CACHE_MAX = 128
_PLAN_CACHE: "OrderedDict" = OrderedDict()
_PLAN_LOCK = threading.Lock()


def get_plan(bg, rows_used: int, cfg: DecodeConfig, device: int = 0, coscheduled: bool = False) -> Plan:
    key = (str(bg.id).upper(), int(bg.z), int(rows_used), _graph_fingerprint(bg, rows_used),
           cfg.precision, float(cfg.beta), int(cfg.max_iter), cfg.early_stop, cfg.crc_kind, device,
           bool(coscheduled))
    with _PLAN_LOCK:
        plan = _PLAN_CACHE.get(key)
        if plan is None:
            plan = Plan(bg, rows_used, cfg, device, coscheduled)
            _PLAN_CACHE[key] = plan
            while len(_PLAN_CACHE) > max(1, PLAN_CACHE_MAX):
                _PLAN_CACHE.popitem(last=False)
        else:
            _PLAN_CACHE.move_to_end(key)
        return plan


def _graph_fingerprint(bg, rows_used: int) -> int:
    cached = getattr(bg, "__dict__", {}).get("_nrldpc_fp")
    if cached is not None and cached[0] == rows_used:
        return cached[1]
    t = edge_tables(bg, rows_used)
    fp = hash((t.row_start.tobytes(), t.cols.tobytes(), t.shifts.tobytes()))
    try:
        bg.__dict__["_nrldpc_fp"] = (rows_used, fp)
    except (AttributeError, TypeError):
        pass
    return fp


def unpack_bits(words: np.ndarray, k: int) -> np.ndarray:
    """(B, ceil(K/32)) LSB-first uint32 words -> (B, K) uint8 0/1
    (decoder.py:332-334 layout), on the library's host threads."""
    w = np.ascontiguousarray(words).view(np.uint32)
    if w.ndim != 2 or w.shape[1] * 32 < k:
        raise ValueError("unpack_bits needs (B, ceil(K/32)) words")
    out = np.empty((w.shape[0], int(k)), np.uint8)
    _native.check(_native.load().nrldpc_unpack_bits(w.ctypes.data, w.shape[0], w.shape[1], int(k),
                                                    out.ctypes.data))
    return out


def _rows_used(n_c: int, bg) -> int:
    if n_c % bg.z:
        raise ValueError("LLR block length must be a multiple of Z")
    rows_used = n_c // bg.z - bg.k_b
    if not 4 <= rows_used <= bg.m_bg:
        raise ValueError(f"LLR block length implies rows_used={rows_used}, outside [4, {bg.m_bg}]")
    return rows_used


def _is_torch(x) -> bool:
    return type(x).__module__.split(".")[0] == "torch"


def decode(llrs, bg, cfg: DecodeConfig, trace: list | None = None) -> DecodeResult:
    """Layered min-sum decode of one batch of quantized LLR blocks on the GPU.

    Same contract as ldpclab.decoder.decode (decoder.py:543-566): ``llrs`` is
    (n_c,) or (B, n_c); results are host numpy arrays.
    """
    cfg = _coerce_cfg(cfg)
    if _is_torch(llrs) and llrs.is_cuda:
        return _decode_torch(llrs, bg, cfg, trace)
    arr = np.asarray(llrs)
    if arr.ndim == 1:
        arr = arr[None, :]
    if cfg.precision is Precision.INT8 and cfg.rho == 4 and arr.shape[0] % 4:
        raise ValueError("packed int8 decode needs a multiple of 4 codewords")
    rows_used = _rows_used(arr.shape[-1], bg)
    if cfg.precision is Precision.INT8:
        if arr.dtype == np.int8:
            # the only out-of-range int8 value is -128; the decode kernel
            # flags it and the call raises the same ValueError (no result)
            host = np.ascontiguousarray(arr)
        else:
            wide = arr.astype(np.int32)  # decoder.py:286 (astype semantics)
            if wide.size and np.abs(wide).max() > INT8_SAT:
                raise ValueError("int8 LLR magnitudes must be at most 127")
            host = np.ascontiguousarray(wide.astype(np.int8))
    else:
        host = np.ascontiguousarray(arr.astype(_FLOAT_DTYPE[cfg.precision]))
    plan = get_plan(bg, rows_used, cfg)
    if trace is None:
        # host buffers straight through the C ABI's pipelined path (chunked
        # H2D copies overlapped with the decode, one result copy-out)
        batch = int(host.shape[0])
        if batch == 0:
            return _empty_result(plan.k, cfg)
        # pageable arrays are staged through the plan's pinned buffers by the
        # library's host threads, overlapped with the chunks' DMA; the bits
        # come back as (B, K) bytes, unpacked chunk by chunk in the pipeline
        out = plan.decode_host_bytes(host, chunks=max(1, min(12, batch // 86)))
        return DecodeResult(
            bits=out["bits"],
            iterations=out["iters"].astype(np.int64),
            success=out["success"].astype(bool),
            syndrome_weight=out["synd"].astype(np.int64),
            crc_ok=out["crc_ok"].astype(bool) if cfg.early_stop is EarlyStop.CRC else None,
        )
    import torch
    dev_in = torch.from_numpy(host).to(f"cuda:{plan.device}", non_blocking=False)
    return _run(plan, dev_in, cfg, trace)


def _empty_result(k: int, cfg: DecodeConfig) -> DecodeResult:
    return DecodeResult(bits=np.zeros((0, k), np.uint8), iterations=np.zeros(0, np.int64),
                        success=np.zeros(0, bool), syndrome_weight=np.zeros(0, np.int64),
                        crc_ok=np.zeros(0, bool) if cfg.early_stop is EarlyStop.CRC else None)


def _decode_torch(llrs, bg, cfg, trace):
    x = llrs
    if x.dim() == 1:
        x = x.unsqueeze(0)
    if cfg.rho == 4 and x.shape[0] % 4:
        raise ValueError("packed int8 decode needs a multiple of 4 codewords")
    rows_used = _rows_used(int(x.shape[-1]), bg)
    import torch
    if cfg.precision is not Precision.INT8:
        x = x.to(torch.float16 if cfg.precision is Precision.F16 else torch.float32)
    elif x.dtype != torch.int8:
        wide = x.to(torch.int32)
        if wide.numel() and int(wide.abs().max()) > INT8_SAT:
            raise ValueError("int8 LLR magnitudes must be at most 127")
        x = wide.to(torch.int8)
    plan = get_plan(bg, rows_used, cfg, device=x.device.index or 0)
    return _run(plan, x.contiguous(), cfg, trace)


def _run(plan: Plan, dev_in, cfg: DecodeConfig, trace, flooding: bool = False) -> DecodeResult:
    import torch
    batch = int(dev_in.shape[0])
    k = plan.k
    if batch == 0:
        return _empty_result(k, cfg)
    out = plan.alloc_outputs(batch, trace=trace is not None)
    if flooding:
        plan.decode_flooding_device(dev_in, out)
    else:
        plan.decode_device(dev_in, out)
    host = {name: t.cpu().numpy() for name, t in out.items()}  # synchronizes
    if int(host["status"][0]):
        raise ValueError("int8 LLR magnitudes must be at most 127")
    iterations = host["iters"].astype(np.int64)
    res = DecodeResult(
        bits=unpack_bits(host["bits"], k),
        iterations=iterations,
        success=host["success"].astype(bool),
        syndrome_weight=host["synd"].astype(np.int64),
        crc_ok=host["crc_ok"].astype(bool) if cfg.early_stop is EarlyStop.CRC else None,
    )
    if trace is not None:
        _append_trace(trace, host["trace_w"], host["trace_m"], iterations, cfg)
    del torch
    return res


def _append_trace(trace: list, tw: np.ndarray, tm: np.ndarray, iterations: np.ndarray,
                  cfg: DecodeConfig) -> None:
    """Rebuild the reference's trace order (decoder.py:497-503, 558-564).

    Every codeword ran max_iter iterations on the device; the reference's batch
    loop stops once all of its codewords are done, i.e. after
    max(iterations) iterations, and rho=4 runs groups of four separately.
    """
    batch = len(iterations)
    group = 4 if (cfg.precision is Precision.INT8 and cfg.rho == 4) else batch
    for g0 in range(0, batch, group):
        members = range(g0, min(g0 + group, batch))
        last = int(iterations[g0:g0 + group].max())
        for it in range(1, last + 1):
            for b in members:
                trace.append((b, it, int(tw[b, it - 1]), float(tm[b, it - 1])))


def decode_flooding(llrs, bg, cfg: DecodeConfig, trace: list | None = None) -> DecodeResult:
    """Flooding-schedule decode on the GPU (decoder.py:569-581): all rows
    consume the previous iteration's posteriors. Same inputs/outputs as
    ``decode``; the packed rho=4 engine is rejected as in the reference."""
    cfg = _coerce_cfg(cfg)
    if cfg.precision is Precision.INT8 and cfg.rho == 4:
        raise ValueError("flooding decoding runs on the scalar path (rho < 4)")
    import torch
    if _is_torch(llrs) and llrs.is_cuda:
        x = llrs.unsqueeze(0) if llrs.dim() == 1 else llrs
        arr = None
    else:
        arr = np.asarray(llrs)
        if arr.ndim == 1:
            arr = arr[None, :]
    n_c = int((x if arr is None else arr).shape[-1])
    rows_used = _rows_used(n_c, bg)
    if arr is not None:
        if cfg.precision is Precision.INT8:
            wide = arr.astype(np.int32)
            if wide.size and np.abs(wide).max() > INT8_SAT:
                raise ValueError("int8 LLR magnitudes must be at most 127")
            arr = wide.astype(np.int8)
        else:
            arr = arr.astype(_FLOAT_DTYPE[cfg.precision])
        plan = get_plan(bg, rows_used, cfg)
        x = torch.from_numpy(np.ascontiguousarray(arr)).to(f"cuda:{plan.device}")
    else:
        if cfg.precision is Precision.INT8:
            if x.dtype != torch.int8:
                wide = x.to(torch.int32)
                if wide.numel() and int(wide.abs().max()) > INT8_SAT:
                    raise ValueError("int8 LLR magnitudes must be at most 127")
                x = wide
            x = x.to(torch.int8)  # an int8 -128 is flagged by the kernel (status word)
        else:
            x = x.to(torch.float16 if cfg.precision is Precision.F16 else torch.float32)
        plan = get_plan(bg, rows_used, cfg, device=x.device.index or 0)
    return _run(plan, x.contiguous(), cfg, trace, flooding=True)


def _coerce_cfg(cfg) -> DecodeConfig:
    if isinstance(cfg, DecodeConfig):
        return cfg
    # the reference's DecodeConfig (same fields): re-validate through ours
    return DecodeConfig(beta=cfg.beta, max_iter=cfg.max_iter, strategy=_enum_value(cfg.strategy),
                        alpha=cfg.alpha, rho=cfg.rho, precision=_enum_value(cfg.precision),
                        early_stop=_enum_value(cfg.early_stop), crc_kind=cfg.crc_kind)
