"""ctypes binding of the C ABI declared in include/nrldpc.h.

This is the only way the package reaches the GPU. There is no CPU fallback:
if ``libnrldpc.so`` is missing or CUDA is unavailable, every decode raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("NRLDPC_LIB", _HERE / "libnrldpc.so"))

NRLDPC_OK = 0
NRLDPC_EINVAL = -1
NRLDPC_ECUDA = -2
NRLDPC_ENOMEM = -3

INT8, F16, F32 = 0, 1, 2
STOP_SYNDROME, STOP_CRC, STOP_NONE = 0, 1, 2
CRC_KINDS = {"crc24a": 0, "crc24b": 1, "crc16": 2}
IN_F64, IN_F32 = 0, 1
MULTI_MAX = 5  # NRLDPC_MULTI_MAX

# every symbol include/nrldpc.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "nrldpc_plan_create",
    "nrldpc_plan_destroy",
    "nrldpc_plan_set_coscheduled",
    "nrldpc_plan_info",
    "nrldpc_quantize",
    "nrldpc_demap_quantize",
    "nrldpc_decode",
    "nrldpc_decode_host",
    "nrldpc_decode_host_bytes",
    "nrldpc_decode_host_async",
    "nrldpc_host_wait",
    "nrldpc_decode_flooding",
    "nrldpc_plan_kernel",
    "nrldpc_decode_multi",
    "nrldpc_encode",
    "nrldpc_channel_awgn",
    "nrldpc_unpack_bits",
    "nrldpc_launch_count",
    "nrldpc_alu_peak",
    "nrldpc_beta_rule",
    "nrldpc_last_error",
)

_lib = None

c_void_p = ctypes.c_void_p
c_int = ctypes.c_int
c_int64 = ctypes.c_int64
c_double = ctypes.c_double


class NativeError(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    """Load libnrldpc.so once; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.is_file():
        raise NativeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the decoder)")
    lib = ctypes.CDLL(str(LIB_PATH))
    lib.nrldpc_plan_create.argtypes = [
        c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, c_int, c_double, c_int, c_int,
        c_int, ctypes.POINTER(c_void_p)]
    lib.nrldpc_plan_create.restype = c_int
    lib.nrldpc_plan_destroy.argtypes = [c_void_p]
    lib.nrldpc_plan_destroy.restype = c_int
    lib.nrldpc_plan_set_coscheduled.argtypes = [c_void_p, c_int]
    lib.nrldpc_plan_set_coscheduled.restype = c_int
    lib.nrldpc_plan_info.argtypes = [c_void_p] + [c_void_p] * 8
    lib.nrldpc_plan_info.restype = c_int
    lib.nrldpc_quantize.argtypes = [c_void_p, c_void_p, c_int, c_int64, c_double, c_double, c_void_p,
                                    c_int, c_void_p]
    lib.nrldpc_quantize.restype = c_int
    lib.nrldpc_demap_quantize.argtypes = [c_void_p, c_void_p, c_int, c_int64, c_double, c_double,
                                          c_double, c_void_p, c_int, c_void_p]
    lib.nrldpc_demap_quantize.restype = c_int
    lib.nrldpc_decode.argtypes = [c_void_p, c_void_p, c_int64] + [c_void_p] * 8 + [c_void_p]
    lib.nrldpc_decode.restype = c_int
    lib.nrldpc_decode_host.argtypes = [c_void_p, c_void_p, c_int64] + [c_void_p] * 5 + [c_int]
    lib.nrldpc_decode_host.restype = c_int
    lib.nrldpc_decode_host_bytes.argtypes = [c_void_p, c_void_p, c_int64] + [c_void_p] * 5 + [c_int]
    lib.nrldpc_decode_host_bytes.restype = c_int
    lib.nrldpc_decode_host_async.argtypes = [c_void_p, c_void_p, c_int64] + [c_void_p] * 5 + [c_int, c_void_p]
    lib.nrldpc_decode_host_async.restype = c_int
    lib.nrldpc_host_wait.argtypes = [c_void_p, c_int64]
    lib.nrldpc_host_wait.restype = c_int
    lib.nrldpc_decode_flooding.argtypes = [c_void_p, c_void_p, c_int64] + [c_void_p] * 9
    lib.nrldpc_decode_flooding.restype = c_int
    lib.nrldpc_plan_kernel.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p]
    lib.nrldpc_plan_kernel.restype = c_int
    lib.nrldpc_decode_multi.argtypes = [c_void_p, c_int, c_void_p, c_void_p] + [c_void_p] * 5 + [c_void_p, c_void_p]
    lib.nrldpc_decode_multi.restype = c_int
    lib.nrldpc_encode.argtypes = [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]
    lib.nrldpc_encode.restype = c_int
    lib.nrldpc_channel_awgn.argtypes = [c_void_p, c_void_p, c_int64, c_double, c_double,
                                        ctypes.c_uint64, c_void_p, c_void_p]
    lib.nrldpc_channel_awgn.restype = c_int
    lib.nrldpc_alu_peak.argtypes = [c_int, c_void_p, c_void_p]
    lib.nrldpc_alu_peak.restype = c_int
    lib.nrldpc_beta_rule.argtypes = [c_double, c_void_p, c_void_p, c_void_p, c_void_p]
    lib.nrldpc_beta_rule.restype = c_int
    lib.nrldpc_unpack_bits.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_void_p]
    lib.nrldpc_unpack_bits.restype = c_int
    lib.nrldpc_launch_count.argtypes = []
    lib.nrldpc_launch_count.restype = c_int
    lib.nrldpc_last_error.argtypes = []
    lib.nrldpc_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == NRLDPC_OK:
        return
    msg = load().nrldpc_last_error().decode(errors="replace")
    if rc == NRLDPC_EINVAL:
        raise ValueError(msg)
    raise NativeError(f"nrldpc error {rc}: {msg}")


def launch_count() -> int:
    return int(load().nrldpc_launch_count())
