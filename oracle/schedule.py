"""2D Communication Scheduling pieces (oracle; test infrastructure only).

Vertical Sparse Scheduling — Algorithm 1:
    G_coalesced <- COALESCE(G)                       (line 2)
    D_u         <- UNIQUE(D_cur[n])                   (line 3)
    i_prior     <- D_u ∩ D_next                       (line 4)
    i_scheduled <- D_u \\ i_prior                      (line 5)
    G_p <- INDEX_SELECT(G_coalesced, i_prior)         (line 6)
    G_d <- INDEX_SELECT(G_coalesced, i_scheduled)     (line 7)
D_next is the gathered (global) next batch — DESIGN.md reading R1.

Horizontal Scheduling priority queue: "Among the
parameters ready for exchange gradients, the parameter that owns the highest
priority would aggregate gradients first"; dense blocks get priority in FP
dependency order; the prior sparse part gets the highest
priority and the scheduled part the latest.  DESIGN.md reading
R16 makes the issue order a pure function of the enqueue sequence (window W).
"""

import numpy as np

from . import sparse

PRIO_PRIOR = -(2 ** 31)      # "highest communication priority"
PRIO_SCHEDULED = 2 ** 31 - 1  # "the latest"


def vertical_split(G_idx, G_val, D_cur, D_next, n):
    """Algorithm 1 verbatim.  ``D_cur`` is the list of per-rank token lists of
    the current iteration (gathered), ``D_next`` the gathered next batch (any
    iterable of ids, may be empty), ``n`` the process rank.
    Returns ((Gp_idx, Gp_val), (Gd_idx, Gd_val), i_prior, i_scheduled)."""
    if n < 0 or n >= len(D_cur):
        raise ValueError(f"rank {n} out of range")
    Gc_idx, Gc_val, _ = sparse.coalesce(G_idx, G_val)                 # line 2
    D_u = set(int(x) for x in np.unique(np.asarray(D_cur[n], dtype=np.int64)))   # line 3
    next_set = set(int(x) for x in np.asarray(list(D_next), dtype=np.int64))
    i_prior = D_u & next_set                                           # line 4
    i_scheduled = D_u - i_prior                                        # line 5
    Gp = sparse.index_select(Gc_idx, Gc_val, i_prior)                  # line 6
    Gd = sparse.index_select(Gc_idx, Gc_val, i_scheduled)              # line 7
    return Gp, Gd, i_prior, i_scheduled


def issue_order(priorities, window):
    """Deterministic priority-queue issue rule (reading R16).

    Requests arrive in list order (seq = position).  After each arrival, while
    the pending set holds >= ``window`` requests, the one with the smallest
    (priority, seq) is issued.  At the end (flush) the rest is issued in
    (priority, seq) order.  window = 1 is FIFO (Default Scheduling,
    PAPER.md:323-325); window >= len(priorities) issues everything in
    priority order.  Returns the issued seq numbers."""
    if window < 1:
        raise ValueError("window must be >= 1")
    pending, out = [], []
    for seq, p in enumerate(priorities):
        pending.append((int(p), seq))
        while len(pending) >= window:
            best = min(pending)
            pending.remove(best)
            out.append(best[1])
    for item in sorted(pending):
        out.append(item[1])
    return out


def prefetch_window(batches):
    """PAPER.md:374 "always keep the data of the next iteration in memory":
    yields (current, next) with next = None for the final batch (reading R8:
    then D_next is empty and everything is scheduled)."""
    batches = list(batches)
    for i, b in enumerate(batches):
        yield b, (batches[i + 1] if i + 1 < len(batches) else None)
