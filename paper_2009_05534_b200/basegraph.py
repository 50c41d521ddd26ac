"""Quasi-cyclic base graphs (BG1/BG2) and their per-Z lifted edge tables.

Host-side mirror of the reference's graph layer
(/root/reference/pkg/src/ldpclab/basegraph.py): same lifting sets
(basegraph.py:22-35), same shift-column selection and mod-Z reduction
(basegraph.py:125-144), same validation messages (basegraph.py:51,111,130-158),
same ``row_entries`` contract (ascending column, basegraph.py:79-82) and the
same ``code_params`` arithmetic (basegraph.py:222-236).

The shift tables are the reference's synthetic assets, re-encoded losslessly
into ``assets/basegraphs.npz`` by ``tools/make_assets.py`` (the source CSV
sha256 is kept in ``assets/provenance.json`` and checked by the tests).

The decode kernels never see this class: ``LiftedGraph.edge_tables`` flattens
the first ``rows_used`` rows into the (row_start, col, shift) arrays that the
C-ABI plan copies into kernel parameters.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass, field
from fractions import Fraction
from pathlib import Path

import numpy as np

LIFTING_SETS: tuple[tuple[int, ...], ...] = (
    (2, 4, 8, 16, 32, 64, 128, 256),
    (3, 6, 12, 24, 48, 96, 192, 384),
    (5, 10, 20, 40, 80, 160, 320),
    (7, 14, 28, 56, 112, 224),
    (9, 18, 36, 72, 144, 288),
    (11, 22, 44, 88, 176, 352),
    (13, 26, 52, 104, 208),
    (15, 30, 60, 120, 240),
)

ALL_LIFTING_SIZES: tuple[int, ...] = tuple(sorted(z for s in LIFTING_SETS for z in s))

# graph id -> (k_b, m_bg, n_cols, entries)
GRAPH_DIMS = {"BG1": (22, 46, 68, 316), "BG2": (10, 42, 52, 197)}

_ASSET = Path(__file__).resolve().parent / "assets" / "basegraphs.npz"


def lifting_set_index(z: int) -> int:
    """Index of the lifting set holding ``z`` (selects the shift column)."""
    for i, zs in enumerate(LIFTING_SETS):
        if z in zs:
            return i
    raise ValueError(f"Z={z} is not a valid lifting size (a*2^j, a in "
                     f"{{2,3,5,7,9,11,13,15}}, Z <= 384)")


def normalize_id(bg_id) -> str:
    if isinstance(bg_id, (int, np.integer)):
        bg_id = f"BG{int(bg_id)}"
    name = str(bg_id).upper()
    if name not in GRAPH_DIMS:
        raise ValueError(f"unknown base graph id {name!r} (expected BG1 or BG2)")
    return name


@functools.lru_cache(maxsize=None)
def _raw_tables(name: str):
    with np.load(_ASSET) as npz:
        key = name.lower()
        return (npz[f"{key}_rows"].astype(np.int64),
                npz[f"{key}_cols"].astype(np.int64),
                npz[f"{key}_shifts"].astype(np.int64))


@dataclass(frozen=True)
class BaseGraph:
    """A base graph lifted to one Z: entries sorted by (row, col), shifts mod Z."""

    id: str
    k_b: int
    m_bg: int
    n_cols: int
    z: int
    rows: np.ndarray
    cols: np.ndarray
    shifts: np.ndarray
    w_r: np.ndarray = field(repr=False)
    w_c: np.ndarray = field(repr=False)
    row_start: np.ndarray = field(repr=False)
    core_sum_shift: int = field(repr=False, default=0)

    @property
    def n_entries(self) -> int:
        return int(len(self.rows))

    @property
    def core_parity_col(self) -> int:
        return self.k_b

    def row_entries(self, r: int) -> tuple[np.ndarray, np.ndarray]:
        lo, hi = int(self.row_start[r]), int(self.row_start[r + 1])
        return self.cols[lo:hi], self.shifts[lo:hi]


def load_basegraph(bg_id, z: int) -> BaseGraph:
    """Lift ``bg_id`` to ``z`` exactly as the reference loader does."""
    name = normalize_id(bg_id)
    set_idx = lifting_set_index(int(z))
    k_b, m_bg, n_cols, n_entries = GRAPH_DIMS[name]
    rows, cols, raw_shifts = _raw_tables(name)
    if len(rows) != n_entries:
        raise ValueError(f"malformed asset: expected {n_entries} entries, got {len(rows)}")
    shifts = np.mod(raw_shifts[:, set_idx], z).astype(np.int64)
    order = np.lexsort((cols, rows))
    rows, cols, shifts = rows[order], cols[order], shifts[order]
    keys = rows * n_cols + cols
    if len(np.unique(keys)) != len(keys):
        raise ValueError("malformed asset: duplicate (row, col) entries")
    if rows.min() < 0 or rows.max() >= m_bg or cols.min() < 0 or cols.max() >= n_cols:
        raise ValueError("malformed asset: entry index out of range")
    w_r = np.bincount(rows, minlength=m_bg)
    w_c = np.bincount(cols, minlength=n_cols)
    if w_r.min() < 3:
        raise ValueError("malformed asset: base row with weight < 3")
    row_start = np.concatenate([[0], np.cumsum(w_r)]).astype(np.int64)
    for a in (rows, cols, shifts, w_r, w_c, row_start):
        a.flags.writeable = False
    bg = BaseGraph(id=name, k_b=k_b, m_bg=m_bg, n_cols=n_cols, z=int(z),
                   rows=rows, cols=cols, shifts=shifts, w_r=w_r, w_c=w_c,
                   row_start=row_start)
    object.__setattr__(bg, "core_sum_shift", _core_sum_shift(bg))
    return bg


def _core_sum_shift(bg: BaseGraph) -> int:
    """Shift of the single circulant left at the first parity column when the
    four core rows are XORed (the systematic encoder solves it first).
    Same structural checks as the reference (basegraph.py:175-207)."""
    p0 = bg.core_parity_col
    for r in range(4, bg.m_bg):
        cols, shifts = bg.row_entries(r)
        own = p0 + r
        if own not in cols:
            raise ValueError(f"{bg.id}: row {r} lacks its extension column {own}")
        if shifts[np.searchsorted(cols, own)] != 0:
            raise ValueError(f"{bg.id}: extension column of row {r} is not identity")
        if (cols >= p0 + 4).sum() != 1:
            raise ValueError(f"{bg.id}: row {r} references a later extension column")
    core: dict[int, list[int]] = {c: [] for c in range(p0, p0 + 4)}
    for r in range(4):
        cols, shifts = bg.row_entries(r)
        for c, s in zip(cols.tolist(), shifts.tolist()):
            if p0 <= c < p0 + 4:
                core[c].append(s)
    for c in range(p0 + 1, p0 + 4):
        if len(core[c]) % 2 or len(set(core[c])) > 1:
            raise ValueError(f"{bg.id}: core rows do not cancel at column {c}")
    odd = [s for s in set(core[p0]) if core[p0].count(s) % 2 == 1]
    if len(odd) != 1:
        raise ValueError(f"{bg.id}: core rows do not sum to a single circulant at column {p0}")
    return int(odd[0])


@dataclass(frozen=True)
class CodeParams:
    z: int
    k: int
    n_c: int
    n_tx: int
    rate: Fraction
    rows_used: int


def code_params(bg, z: int, rows_used: int) -> CodeParams:
    if z != bg.z:
        raise ValueError(f"graph was lifted for Z={bg.z}, not Z={z}")
    if not 4 <= rows_used <= bg.m_bg:
        raise ValueError(
            f"rows_used must be in [4, {bg.m_bg}] (first four rows form the "
            f"parity core), got {rows_used}")
    k = z * bg.k_b
    n_c = z * (bg.k_b + rows_used)
    return CodeParams(z=z, k=k, n_c=n_c, n_tx=n_c - 2 * z,
                      rate=Fraction(k, n_c), rows_used=rows_used)


@dataclass(frozen=True)
class EdgeTables:
    """Flattened layered schedule for (graph, Z, rows_used): the plan input."""

    graph: str
    k_b: int
    z: int
    rows_used: int
    row_start: np.ndarray   # int32 (rows_used + 1,)
    cols: np.ndarray        # int16 (E,)
    shifts: np.ndarray      # int16 (E,), already mod Z

    @property
    def n_edges(self) -> int:
        return int(self.row_start[-1])

    @property
    def n_blocks(self) -> int:
        return self.k_b + self.rows_used


def edge_tables(bg, rows_used: int) -> EdgeTables:
    """Flatten rows 0..rows_used-1 of any BaseGraph-like object (ours or the
    reference's ``ldpclab.BaseGraph``: only ``row_entries``/``k_b``/``z``/``id``
    are used)."""
    starts = [0]
    cols, shifts = [], []
    for r in range(rows_used):
        c, s = bg.row_entries(r)
        cols.append(np.asarray(c, dtype=np.int64))
        shifts.append(np.asarray(s, dtype=np.int64) % bg.z)
        starts.append(starts[-1] + len(c))
    return EdgeTables(
        graph=normalize_id(bg.id), k_b=int(bg.k_b), z=int(bg.z), rows_used=int(rows_used),
        row_start=np.asarray(starts, dtype=np.int32),
        cols=np.concatenate(cols).astype(np.int16),
        shifts=np.concatenate(shifts).astype(np.int16),
    )
