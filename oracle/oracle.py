"""Python wrapper of the C oracle (ldpc_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg, never by the product package. It restates
ldpclab.decoder.decode (/root/reference/pkg/src/ldpclab/decoder.py:486-566)
on the CPU and returns the same fields; it is pinned against golden vectors
produced by the reference itself (tests/golden/, tests/test_oracle.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libldpc_oracle.so"

PREC = {"int8": 0, "f16": 1, "f32": 2}
STOP = {"syndrome": 0, "crc": 1, "none": 2}
CRC = {"crc24a": (24, 0x864CFB), "crc24b": (24, 0x800063), "crc16": (16, 0x1021)}

_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not LIB.is_file():
            build()
        lib = ctypes.CDLL(str(LIB))
        vp = ctypes.c_void_p
        lib.oracle_decode.argtypes = [
            ctypes.c_int, vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp,
            ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint32,
            vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int]
        lib.oracle_decode.restype = ctypes.c_int
        lib.oracle_quantize_i8.argtypes = [vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_double, vp]
        lib.oracle_quantize_i8.restype = None
        _lib = lib
    return _lib


def _val(x):
    return getattr(x, "value", x)


def graph_tables(bg, rows_used: int):
    starts, cols, shifts = [0], [], []
    for r in range(rows_used):
        c, s = bg.row_entries(r)
        cols.extend(int(v) for v in c)
        shifts.extend(int(v) % bg.z for v in s)
        starts.append(len(cols))
    return (np.asarray(starts, np.int32), np.asarray(cols, np.int16), np.asarray(shifts, np.int16))


def decode_flooding(llrs, bg, cfg, trace: list | None = None, threads: int = 0) -> dict:
    """Flooding schedule (decoder.py:337-365, 569-581)."""
    return decode(llrs, bg, cfg, trace, threads, flooding=True)


def decode(llrs, bg, cfg, trace: list | None = None, threads: int = 0, flooding: bool = False) -> dict:
    """Oracle decode. ``cfg`` is any DecodeConfig-like object (ours or the
    reference's). Returns a dict with bits/iterations/success/syndrome_weight/
    crc_ok and, when ``trace`` is a list, appends the reference-ordered trace."""
    lib = _load()
    prec = str(_val(cfg.precision))
    stop = str(_val(cfg.early_stop))
    arr = np.asarray(llrs)
    if arr.ndim == 1:
        arr = arr[None, :]
    dtype = {"int8": np.int8, "f16": np.float16, "f32": np.float32}[prec]
    if prec == "int8":
        wide = arr.astype(np.int32)
        if wide.size and np.abs(wide).max() > 127:
            raise ValueError("int8 LLR magnitudes must be at most 127")
        arr = wide.astype(np.int8)
    arr = np.ascontiguousarray(arr.astype(dtype, copy=False))
    b, n_c = arr.shape
    if n_c % bg.z:
        raise ValueError("LLR block length must be a multiple of Z")
    rows_used = n_c // bg.z - bg.k_b
    if not 4 <= rows_used <= bg.m_bg:
        raise ValueError(f"LLR block length implies rows_used={rows_used}, outside [4, {bg.m_bg}]")
    rs, cols, shifts = graph_tables(bg, rows_used)
    k = bg.k_b * bg.z
    crc_len, crc_poly = CRC[cfg.crc_kind]
    bits = np.zeros((b, k), np.uint8)
    iters = np.zeros(b, np.int64)
    synd = np.zeros(b, np.int64)
    success = np.zeros(b, np.uint8)
    crc_ok = np.zeros(b, np.uint8)
    tw = np.zeros((b, cfg.max_iter), np.int32) if trace is not None else None
    tm = np.zeros((b, cfg.max_iter), np.float64) if trace is not None else None
    rc = lib.oracle_decode(
        PREC[prec], arr.ctypes.data, b, bg.k_b, bg.z, rows_used, rs.ctypes.data, cols.ctypes.data,
        shifts.ctypes.data, float(cfg.beta), int(cfg.max_iter), STOP[stop], crc_len, crc_poly,
        bits.ctypes.data, iters.ctypes.data, synd.ctypes.data, success.ctypes.data, crc_ok.ctypes.data,
        tw.ctypes.data if tw is not None else None, tm.ctypes.data if tm is not None else None,
        int(threads or os.cpu_count() or 1), int(flooding))
    if rc:
        raise MemoryError("oracle workspace allocation failed")
    out = {"bits": bits, "iterations": iters, "success": success.astype(bool),
           "syndrome_weight": synd, "crc_ok": crc_ok.astype(bool) if stop == "crc" else None}
    if trace is not None:
        group = 4 if (prec == "int8" and int(cfg.rho) == 4) else b
        for g0 in range(0, b, group):
            last = int(iters[g0:g0 + group].max())
            for it in range(1, last + 1):
                for i in range(g0, min(g0 + group, b)):
                    trace.append((i, it, int(tw[i, it - 1]), float(tm[i, it - 1])))
    return out


def quantize_i8(llr: np.ndarray, z: int, scale: float = 8.0) -> np.ndarray:
    """channel.quantize int8 mode (channel.py:64-83) on the CPU."""
    lib = _load()
    x = np.ascontiguousarray(np.asarray(llr, dtype=np.float64))
    lead = x.shape[:-1]
    x2 = x.reshape(-1, x.shape[-1])
    out = np.empty((x2.shape[0], x2.shape[1] + 2 * z), np.int8)
    lib.oracle_quantize_i8(x2.ctypes.data, x2.shape[0], x2.shape[1], 2 * z, float(scale),
                           out.ctypes.data)
    return out.reshape(lead + (out.shape[-1],))
