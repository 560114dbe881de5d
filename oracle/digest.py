"""Content digests for full-size parity (TEST INFRASTRUCTURE -- never imported by the
product package).

The BASELINE configurations are too large to commit as fixtures (the 1080p 4-bounce
frame alone is 8,184,972 vertices), so `tests/golden/make_fullsize.py` runs the
reference on them here and commits SHA-256 digests of its outputs
(`tests/golden/fullsize.json`); the `-m gpu` tests digest the device results the same
way.  Every digest covers dtype, shape and the raw bytes, so equal digests mean
bit-identical arrays.

Tables are compared order-free (`table_digest`): the parallel insert may place keys
that compete for one probe window in a different slot than the reference's sequential
scan (src/_native.pyx:209-247), so a table is digested as the sorted list of its
occupied rows -- tag, live / history counts, last_touch, sums, history sums, delta --
which is exactly the per-key content the reference's tables hold.
"""

from __future__ import annotations

import hashlib

import numpy as np

EMPTY = np.uint64(0xFFFFFFFF00000000)
TABLE_FIELDS = ("tags", "sums", "counts", "hist_sums", "hist_counts", "last_touch", "deltas")


def digest(a) -> str:
    """SHA-256 (32 hex digits) of an array's dtype, shape and C-order bytes."""
    a = np.ascontiguousarray(np.asarray(a))
    h = hashlib.sha256()
    h.update(f"{a.dtype.str}|{a.shape}|".encode())
    h.update(memoryview(a).cast("B"))
    return h.hexdigest()[:32]


def _bits(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a))
    return a.view(np.int64) if a.dtype.itemsize == 8 else a.astype(np.int64)


def table_rows(st: dict) -> np.ndarray:
    """Occupied rows of a table state as int64 columns (tag, counts, hist_counts,
    last_touch, sums x3, hist_sums x3, deltas), sorted lexicographically."""
    tags = np.asarray(st["tags"]).view(np.uint64)
    occ = np.nonzero(tags != EMPTY)[0]
    cols = [tags[occ].view(np.int64), _bits(st["counts"])[occ], _bits(st["hist_counts"])[occ],
            _bits(st["last_touch"])[occ]]
    sums, hist = _bits(st["sums"]).reshape(-1, 3), _bits(st["hist_sums"]).reshape(-1, 3)
    cols += [sums[occ, c] for c in range(3)] + [hist[occ, c] for c in range(3)]
    cols.append(_bits(st["deltas"])[occ])
    rows = np.stack(cols, axis=1) if len(occ) else np.zeros((0, 11), np.int64)
    order = np.lexsort(rows.T[::-1]) if len(rows) else np.zeros(0, np.int64)
    return np.ascontiguousarray(rows[order])


def table_digest(st: dict) -> dict:
    rows = table_rows(st)
    return {"occupied": int(len(rows)), "rows": digest(rows),
            "counts": int(np.asarray(st["counts"]).sum()),
            "hist_counts": int(np.asarray(st["hist_counts"]).sum())}


def composite(base: np.ndarray, pixel: np.ndarray, throughput: np.ndarray, chosen: np.ndarray,
              spp: int) -> np.ndarray:
    """The reference's composite (src/pipeline.py:280-282): np.add.at in vertex order,
    then base + flat / spp."""
    h, w = base.shape[:2]
    flat = np.zeros((h * w, 3))
    np.add.at(flat, pixel, throughput * chosen)
    return base + flat.reshape(h, w, 3) / spp
