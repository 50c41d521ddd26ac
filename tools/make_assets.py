"""Re-encode the reference base-graph tables into the package's npz asset.

The decoder's parity depends on the reference's *synthetic* shift tables
(/root/reference/pkg/src/ldpclab/assets/{bg1,bg2}.csv, sha256-pinned in
assets/manifest.json there). They are data, not code; this script stores
them as integer arrays (rows, cols, shift columns s0..s7) and records the
sha256 of each source CSV so tests can prove the re-encoding is lossless.

Run in the build container only (needs /root/reference):
    python tools/make_assets.py
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

SRC = Path("/root/reference/pkg/src/ldpclab/assets")
DST = Path(__file__).resolve().parents[1] / "paper_2009_05534_b200" / "assets"


def main() -> int:
    DST.mkdir(parents=True, exist_ok=True)
    arrays = {}
    meta = {}
    for name in ("bg1", "bg2"):
        path = SRC / f"{name}.csv"
        blob = path.read_bytes()
        raw = np.loadtxt(path, dtype=np.int64, delimiter=",", skiprows=1, ndmin=2)
        arrays[f"{name}_rows"] = raw[:, 0].astype(np.int16)
        arrays[f"{name}_cols"] = raw[:, 1].astype(np.int16)
        arrays[f"{name}_shifts"] = raw[:, 2:].astype(np.int16)
        meta[name] = {"source_sha256": hashlib.sha256(blob).hexdigest(),
                      "entries": int(raw.shape[0])}
    np.savez_compressed(DST / "basegraphs.npz", **arrays)
    (DST / "provenance.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print(json.dumps(meta, indent=1))
    return 0


if __name__ == "__main__":
    sys.exit(main())
