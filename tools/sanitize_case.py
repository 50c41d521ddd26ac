#!/usr/bin/env python
"""Small decodes for compute-sanitizer runs (tests/test_gpu_sanitizer.py).

Each case decodes a few codewords through the C ABI and compares with the
oracle, so a sanitizer run also checks the results it instruments. Cases:
  pair    byte-pair layout, several groups per CTA (BG2 Z=64, BG1 Z=20)
  tm      TM layout (shared + tensor memory messages), register rows (BG1 Z=384)
  refill  lane-refill kernel, syndrome stop (BG1 Z=384, BG2 Z=256)
  float   f16 / f32 engines (BG1 Z=384 on chip, BG2 Z=52 workspace)
  quant   quantize + demap kernels, encoder, flooding
"""

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2009_05534_b200 as nr  # noqa: E402
from paper_2009_05534_b200.synth import noisy_llrs  # noqa: E402
from oracle import oracle  # noqa: E402


def check(bg_id, z, rows, n, cfg, ebn0=1.5, prec="int8"):
    bg = nr.load_basegraph(bg_id, z)
    params = nr.code_params(bg, z, rows)
    _, llr = noisy_llrs(bg, rows, ebn0, n, seed=(z, n))
    blocks = nr.quantize(llr, nr.QuantConfig(mode=prec), params)
    res = nr.decode(torch.from_numpy(blocks).cuda(), bg, cfg)
    ref = oracle.decode(blocks, bg, cfg)
    assert np.array_equal(res.bits, ref["bits"]), (bg_id, z, prec)
    assert np.array_equal(res.iterations, ref["iterations"]), (bg_id, z, prec)


def main(which):
    fixed = nr.DecodeConfig(max_iter=2, early_stop="none")
    stop = nr.DecodeConfig(max_iter=4, early_stop="syndrome")
    if "pair" in which:
        check("BG2", 64, 42, 5, fixed)
        check("BG1", 20, 46, 3, stop)
    if "tm" in which:
        check("BG1", 384, 46, 3, fixed)
        check("BG2", 384, 42, 2, fixed)
    if "refill" in which:
        check("BG1", 384, 46, 5, stop, ebn0=2.5)
        check("BG2", 256, 42, 5, stop, ebn0=1.0)
    if "float" in which:
        check("BG1", 384, 46, 2, nr.DecodeConfig(max_iter=2, early_stop="none", precision="f16"), prec="f16")
        check("BG2", 52, 42, 3, nr.DecodeConfig(max_iter=3, precision="f32"), prec="f32")
    if "quant" in which:
        bg = nr.load_basegraph("BG1", 96)
        params = nr.code_params(bg, 96, 46)
        _, llr = noisy_llrs(bg, 46, 2.0, 3, seed=1)
        q = nr.quantize(torch.from_numpy(llr).cuda(), nr.QuantConfig(), params)
        assert np.array_equal(q.cpu().numpy(), oracle.quantize_i8(llr, 96))
        fl = nr.decode_flooding(q, bg, nr.DecodeConfig(max_iter=3))
        assert fl.bits.shape == (3, params.k)
    torch.cuda.synchronize()
    print("sanitize cases ok:", ",".join(which))


if __name__ == "__main__":
    from paper_2009_05534_b200 import _native
    print("library:", _native.LIB_PATH.name)
    main(sys.argv[1:] or ["pair", "tm", "refill", "float", "quant"])
