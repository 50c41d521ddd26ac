"""compute-sanitizer over the CUDA kernels (sanitizers).

memcheck and synccheck over every kernel family (byte-pair, TM with tensor
memory, lane refill, float engines, quantize/flooding); racecheck over the
shared-memory layouts with NRLDPC_NO_TM=1 (tensor-memory rows are
thread-private: each thread owns its TMEM lane). Each run also checks the
decoded results against the oracle (tools/sanitize_case.py).
"""

import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


def _run(tool, cases, env_extra=None, timeout=900):
    env = dict(os.environ)
    env.update(env_extra or {})
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--target-processes", "all",
           sys.executable, str(ROOT / "tools" / "sanitize_case.py"), *cases]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
    assert "sanitize cases ok" in out


@pytest.mark.parametrize("cases", [["pair", "quant"], ["tm"], ["refill"], ["float"]])
def test_memcheck(cuda_ok, cases):
    _run("memcheck", cases)


@pytest.mark.parametrize("cases", [["pair"], ["tm", "refill"], ["float"]])
def test_synccheck(cuda_ok, cases):
    _run("synccheck", cases)


def test_racecheck_shared_memory_layouts(cuda_ok):
    _run("racecheck", ["pair"], {"NRLDPC_NO_TM": "1"})
