"""Access to the reference-generated golden vectors (tests/golden/)."""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@dataclass
class Case:
    name: str
    bg: str
    z: int
    rows: int
    trace: bool
    cfg: dict
    flooding: bool
    arrays: dict = field(repr=False)

    @property
    def llr(self):
        return self.arrays["llr"]

    def bits(self):
        k = (22 if self.bg == "BG1" else 10) * self.z
        return np.unpackbits(self.arrays["bits"], axis=1, bitorder="little")[:, :k]

    def trace_list(self):
        t = self.arrays["trace"]
        return [(int(c), int(i), int(w), float(m)) for c, i, w, m in t]


@lru_cache(maxsize=1)
def load_cases() -> dict:
    meta = json.loads((GOLDEN / "cases.json").read_text())
    data = np.load(GOLDEN / "golden.npz")
    cases = {}
    for m in meta["cases"]:
        pre = m["name"] + "/"
        arrays = {k[len(pre):]: data[k] for k in data.files if k.startswith(pre)}
        cases[m["name"]] = Case(m["name"], m["bg"], m["z"], m["rows"], m["trace"], m["cfg"],
                                m.get("flooding", False), arrays)
    quant = {k.split("/", 1)[1]: data[k] for k in data.files if k.startswith("quant/")}
    return {"cases": cases, "quant": quant}


def make_cfg(case: Case, cls):
    c = dict(case.cfg)
    return cls(**c)
