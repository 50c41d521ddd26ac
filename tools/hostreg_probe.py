"""Cost of page-locking a caller's pageable buffer in place (cudaHostRegister)
vs copying it into pinned staging memory, for one 26.7 MB batch."""
import ctypes
import time

import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so.12") if False else None
lib = ctypes.CDLL(torch._C.__file__)  # noqa: F841 (torch loaded cudart)
rt = ctypes.CDLL("libcudart.so")
n = 1024 * 26112
for rep in range(5):
    a = np.random.default_rng(rep).integers(-127, 128, size=n, dtype=np.int8)
    t0 = time.perf_counter()
    rc = rt.cudaHostRegister(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(n), 0)
    t1 = time.perf_counter()
    rc2 = rt.cudaHostUnregister(ctypes.c_void_p(a.ctypes.data))
    t2 = time.perf_counter()
    print(f"register {1e3 * (t1 - t0):.3f} ms (rc {rc}), unregister {1e3 * (t2 - t1):.3f} ms (rc {rc2})")
