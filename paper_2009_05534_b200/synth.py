"""Synthetic AWGN traffic (host side), reproducing the reference's generator.

``noisy_llrs`` follows the reference fixture make_noisy_blocks
(/root/reference/pkg/tests/conftest.py:37-49) draw-for-draw: the same numpy
PCG64 stream yields messages, then BPSK + AWGN noise, then L = 2y/sigma^2.
Quantization is left to the GPU (``channel.quantize``), so the returned
float64 LLRs are exactly what the reference would quantize.
"""

from __future__ import annotations

import numpy as np

from .basegraph import code_params
from .channel import bpsk_awgn, demap_llr, ebn0_to_sigma
from .codec import encode_batch


def noisy_llrs(bg, rows_used: int, ebn0_db: float, count: int, seed):
    """(messages (count, K) uint8, channel LLRs (count, n_tx) float64)."""
    params = code_params(bg, bg.z, rows_used)
    rng = np.random.default_rng(seed)
    msgs = rng.integers(0, 2, size=(count, params.k), dtype=np.uint8)
    tx = encode_batch(msgs, bg, bg.z, rows_used)[:, 2 * bg.z:]
    sigma = ebn0_to_sigma(ebn0_db, params.k / params.n_tx)
    llr = demap_llr(bpsk_awgn(tx, sigma, rng), sigma)
    return msgs, llr
