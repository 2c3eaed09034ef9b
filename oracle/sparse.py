"""COO sparse embedding gradients (oracle; test infrastructure only).

PAPER.md:130 (§2.2) — embedding gradients are sparse, stored in COO form
(row index + whole row value).  PAPER.md:349-352 (§4.2.2 "Coalescing
Gradients") — "With padding and reduplicate words, the embedding sparse
gradients would have repeated coordinates in the indices.  The multi-valued
elements could be coalesced into a single value using summation".
Alg. 1 line 2 COALESCE; lines 6-7
INDEX_SELECT.

A sparse gradient here is a pair ``(idx, val)``: ``idx`` int64 [c],
``val`` float64 [c, w] (w = row width).  Duplicates allowed until coalesced.
"""

import numpy as np


def coalesce(idx, val):
    """Alg. 1 line 2: COALESCE(G) — merge duplicate row indices by summation.

    Output indices are unique and ascending; duplicates are summed in their
    original entry (position) order (stable sort keeps that order), in fp64.
    Returns (uidx, uval, seg_start) where seg_start[k] is the first position
    (in the stable-sorted order) of output row k.
    """
    idx = np.asarray(idx, dtype=np.int64)
    val = np.asarray(val, dtype=np.float64)
    if idx.size == 0:
        return idx.copy(), val.reshape(0, val.shape[1] if val.ndim == 2 else 0).copy(), np.zeros(0, np.int64)
    order = np.argsort(idx, kind="stable")
    sidx = idx[order]
    heads = np.flatnonzero(np.r_[True, sidx[1:] != sidx[:-1]])
    uval = np.add.reduceat(val[order], heads, axis=0)
    return sidx[heads], uval, heads


def coalesce_abs(idx, val):
    """Same segmentation as :func:`coalesce` but summing |val| — the
    first-order error magnitude sigma of each coalesced row (SURVEY §8(c)
    comparison metric)."""
    return coalesce(idx, np.abs(np.asarray(val, dtype=np.float64)))


def index_select(uidx, uval, keep):
    """Alg. 1 lines 6-7: INDEX_SELECT(G_coalesced, i) — the rows of a coalesced
    gradient whose index is in ``keep`` (kept in ascending order)."""
    mask = np.isin(uidx, np.asarray(list(keep) if isinstance(keep, (set, frozenset)) else keep, dtype=np.int64))
    return uidx[mask], uval[mask]


def densify(idx, val, rows):
    """Dense [rows, w] matrix with duplicate entries accumulated (plain loop)."""
    idx = np.asarray(idx, dtype=np.int64)
    val = np.asarray(val, dtype=np.float64)
    w = val.shape[1] if val.ndim == 2 else 0
    out = np.zeros((rows, w), dtype=np.float64)
    for i in range(idx.size):
        if idx[i] < 0 or idx[i] >= rows:
            raise IndexError(f"row index {idx[i]} out of range [0, {rows})")
        out[idx[i]] += val[i]
    return out


def scatter_add(target, idx, val, scale):
    """target[idx[i]] += scale * val[i] for every entry (plain loop); returns a copy."""
    out = np.array(target, dtype=np.float64, copy=True)
    val = np.asarray(val, dtype=np.float64)
    if val.ndim == 2 and val.shape[1] != out.shape[1]:
        raise ValueError("shape mismatch")
    for i in range(len(idx)):
        out[idx[i]] += scale * val[i]
    return out
