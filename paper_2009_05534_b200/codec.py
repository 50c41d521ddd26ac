"""Host-side systematic encoder, syndrome and CRC helpers.

These produce *synthetic test traffic* for the decoder (bench inputs, BLER
runs); they are not on the accelerated path. Semantics follow the reference
codec (/root/reference/pkg/src/ldpclab/codec.py):

* variable ``c*Z + i`` is circulant position ``i`` of base column ``c``
  (codec.py:3-5); a shift-``s`` circulant maps output ``i`` to input
  ``(i+s) mod Z`` (codec.py:47-49);
* systematic encoding solves the double-diagonal core first, then every
  extension row through its identity column (codec.py:66-139);
* CRC polynomials and the bit-serial register convention (codec.py:16-20,
  172-213).
"""

from __future__ import annotations

import numpy as np

from .basegraph import code_params

CRC_POLYS = {"crc24a": (24, 0x864CFB), "crc24b": (24, 0x800063), "crc16": (16, 0x1021)}


def _circ(block: np.ndarray, s: int) -> np.ndarray:
    return np.roll(block, -int(s), axis=-1)


def encode_batch(messages, bg, z: int, rows_used: int) -> np.ndarray:
    """(B, K) message bits -> (B, n_c) codeword bits (uint8)."""
    params = code_params(bg, z, rows_used)
    msgs = np.asarray(messages, dtype=np.uint8)
    if msgs.ndim != 2 or msgs.shape[1] != params.k:
        raise ValueError(f"expected messages of shape (B, {params.k})")
    if not np.isin(msgs, (0, 1)).all():
        raise ValueError("bit vector may only contain 0 and 1")
    b = msgs.shape[0]
    p0 = bg.k_b
    x = np.zeros((b, bg.k_b + rows_used, z), dtype=np.uint8)
    x[:, :p0] = msgs.reshape(b, p0, z)
    rows = [tuple(map(np.asarray, bg.row_entries(r))) for r in range(rows_used)]

    # information part of every core row
    info = np.zeros((4, b, z), dtype=np.uint8)
    for r in range(4):
        for c, s in zip(*rows[r]):
            if c < p0:
                info[r] ^= _circ(x[:, c], s)
    core_sum_shift = getattr(bg, "core_sum_shift", None)
    if core_sum_shift is None:
        core_sum_shift = bg.__dict__["core_sum_shift"]
    x[:, p0] = np.roll(info[0] ^ info[1] ^ info[2] ^ info[3], int(core_sum_shift), axis=-1)
    known = {p0}
    pending = [0, 1, 2, 3]
    while pending:
        progressed = False
        for r in list(pending):
            cols, shifts = rows[r]
            unknown = [(c, s) for c, s in zip(cols, shifts) if p0 <= c and c not in known]
            if len(unknown) > 1:
                continue
            acc = info[r].copy()
            for c, s in zip(cols, shifts):
                if p0 <= c and c in known:
                    acc ^= _circ(x[:, c], s)
            if unknown:
                c, s = unknown[0]
                x[:, c] = np.roll(acc, int(s), axis=-1)
                known.add(int(c))
            elif acc.any():
                raise ValueError("singular parity core: asset does not encode systematically")
            pending.remove(r)
            progressed = True
        if not progressed:
            raise ValueError("singular parity core: cannot isolate core columns")
    for r in range(4, rows_used):
        cols, shifts = rows[r]
        acc = np.zeros((b, z), dtype=np.uint8)
        for c, s in zip(cols, shifts):
            if c != p0 + r:
                acc ^= _circ(x[:, c], s)
        x[:, p0 + r] = acc
    bits = x.reshape(b, params.n_c)
    if syndrome_weights(bits, bg, rows_used).any():
        raise ValueError("encoder produced a nonzero syndrome (corrupt asset)")
    return bits


def syndrome_weights(bits, bg, rows_used: int) -> np.ndarray:
    """Unsatisfied parity checks per codeword over rows 0..rows_used-1."""
    arr = np.asarray(bits, dtype=np.uint8)
    blocks = arr.reshape(arr.shape[0], -1, bg.z)
    out = np.zeros(arr.shape[0], dtype=np.int64)
    for r in range(rows_used):
        acc = np.zeros((arr.shape[0], bg.z), dtype=np.uint8)
        for c, s in zip(*bg.row_entries(r)):
            acc ^= _circ(blocks[:, c], s)
        out += acc.sum(axis=-1, dtype=np.int64)
    return out


def _crc_params(kind: str) -> tuple[int, int]:
    try:
        return CRC_POLYS[kind]
    except KeyError:
        raise ValueError(f"unknown CRC kind {kind!r}; choose from {sorted(CRC_POLYS)}")


def crc_remainder(bits, kind: str) -> np.ndarray:
    length, poly = _crc_params(kind)
    reg, top, mask = 0, 1 << (length - 1), (1 << length) - 1
    for bit in np.asarray(bits, dtype=np.uint8).ravel().tolist():
        fb = bool(reg & top) ^ bool(bit)
        reg = ((reg << 1) & mask) ^ (poly if fb else 0)
    return np.array([(reg >> (length - 1 - i)) & 1 for i in range(length)], dtype=np.uint8)


def crc_attach(payload, kind: str = "crc24b", k: int | None = None) -> np.ndarray:
    length, _ = _crc_params(kind)
    bits = np.asarray(payload, dtype=np.uint8).ravel()
    if k is not None and len(bits) + length > k:
        raise ValueError(f"payload of {len(bits)} bits plus {length} CRC bits exceeds K={k}")
    return np.concatenate([bits, crc_remainder(bits, kind)])


def crc_check(bits, kind: str = "crc24b") -> bool:
    length, _ = _crc_params(kind)
    data = np.asarray(bits, dtype=np.uint8).ravel()
    if len(data) < length:
        return False
    return not crc_remainder(data, kind).any()
