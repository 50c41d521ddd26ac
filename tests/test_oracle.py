"""Pin the C oracle against golden vectors produced by the reference itself.

CPU only. Every case in tests/golden/golden.npz was decoded by
ldpclab.decoder.decode (tests/golden/make_golden.py); the oracle must agree
bit-for-bit on bits, iterations, success, syndrome weight, crc_ok and trace.
"""

import numpy as np
import pytest

from oracle import oracle
from paper_2009_05534_b200 import DecodeConfig, load_basegraph
from tests.golden_cases import load_cases, make_cfg

CASES = sorted(load_cases()["cases"])


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_golden(name):
    case = load_cases()["cases"][name]
    bg = load_basegraph(case.bg, case.z)
    cfg = make_cfg(case, DecodeConfig)
    trace = [] if case.trace else None
    got = oracle.decode(case.llr, bg, cfg, trace, threads=4, flooding=case.flooding)
    assert np.array_equal(got["bits"], case.bits())
    assert np.array_equal(got["iterations"], case.arrays["iterations"])
    assert np.array_equal(got["success"], case.arrays["success"].astype(bool))
    assert np.array_equal(got["syndrome_weight"], case.arrays["syndrome_weight"])
    if "crc_ok" in case.arrays:
        assert np.array_equal(got["crc_ok"], case.arrays["crc_ok"].astype(bool))
    else:
        assert got["crc_ok"] is None
    if case.trace:
        assert trace == case.trace_list()


def test_oracle_quantize_matches_reference():
    q = load_cases()["quant"]
    got = oracle.quantize_i8(q["x"], z=16)
    assert np.array_equal(got, q["int8"])


def test_oracle_rejects_out_of_range_int8():
    bg = load_basegraph("BG2", 16)
    bad = np.zeros(832, np.int16)
    bad[5] = -128
    with pytest.raises(ValueError, match="at most 127"):
        oracle.decode(bad, bg, DecodeConfig())
