"""Checked build: device-side bounds checks instead of compute-sanitizer.

compute-sanitizer is closed on this GPU pool, so libnrldpc_checked.so
(csrc/Makefile ``checked``, -DNRLDPC_CHECKED) carries its own checks: every
shared-memory access inside the CTA's dynamic window and naturally aligned,
every gathered posterior inside its group's L array, every message slot
inside its thread's row (shared memory) or column slot (tensor memory, own
lane quarter, below column 512), every result write inside the batch. A
violation traps, which fails the subprocess.

The checked library runs the kernel families on small cases (decoded results
compared with the oracle: tools/sanitize_case.py) and the whole golden-vector
suite.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CHECKED = ROOT / "paper_2009_05534_b200" / "libnrldpc_checked.so"


def _env(extra=None):
    if not CHECKED.is_file():
        pytest.fail(f"{CHECKED} missing: build it with __graft_entry__.build() (make -C csrc checked)")
    env = dict(os.environ)
    env["NRLDPC_LIB"] = str(CHECKED)
    env.update(extra or {})
    return env


@pytest.mark.parametrize("cases,extra", [
    (["pair", "quant"], None), (["tm"], None), (["refill"], None), (["float"], None),
    (["tm", "refill"], {"NRLDPC_NO_TM": "1"}),   # byte-pair layouts of the large shapes
])
def test_checked_build_kernel_families(cuda_ok, cases, extra):
    p = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_case.py"), *cases], cwd=ROOT,
                       env=_env(extra), capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
    assert "sanitize cases ok" in p.stdout


def test_checked_build_golden_suite(cuda_ok):
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                        "tests/test_gpu_decode.py", "-k", "golden or ragged or partial or config3"],
                       cwd=ROOT, env=_env(), capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
    assert " passed" in p.stdout
