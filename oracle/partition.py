"""Column-wise embedding partition (oracle; test infrastructure only).

PAPER.md:271 (§4.1.2) — "Assume we partition an embedding with dimension
[L,D] among N training processes, row-wise approach distributes a [L/N,D]
embedding shard to each worker.  In contrast, column-wise approach divides
the embedding into [L, D/N] slices."
PAPER.md:274 — "each partition will get the same amount of requests".
PAPER.md:280 (§4.1.3) — "embedding in each process firstly looks up all
training data of this step".

The paper assumes N | D.  Reading R7: when it does not, earlier
ranks take the extra column (the GPU path rejects N ∤ D with EMB_ERR_SHAPE).
"""

import numpy as np


def column_ranges(D, N):
    """[(c0, c1)] for every rank r; contiguous, ordered by rank, widths differ
    by at most one (earlier ranks wider)."""
    if N < 1 or N > D:
        raise ValueError(f"infeasible partition: N={N}, D={D}")
    base, rem = divmod(D, N)
    out, c = [], 0
    for r in range(N):
        w = base + (1 if r < rem else 0)
        out.append((c, c + w))
        c += w
    return out


def partition_columnwise(W, N):
    """shard_r = W[:, c0_r:c1_r]."""
    W = np.asarray(W)
    return [W[:, c0:c1].copy() for (c0, c1) in column_ranges(W.shape[1], N)]


def row_ranges(L, N):
    """Row-wise comparison partition [L/N, D]; remainder to
    earlier ranks."""
    if N < 1 or N > L:
        raise ValueError(f"infeasible partition: N={N}, L={L}")
    base, rem = divmod(L, N)
    out, c = [], 0
    for r in range(N):
        w = base + (1 if r < rem else 0)
        out.append((c, c + w))
        c += w
    return out


def shard_lookup(shard, tokens):
    """Rows of one column shard for a token list; bounds-checked."""
    tokens = np.asarray(tokens, dtype=np.int64)
    L = shard.shape[0]
    if tokens.size and (tokens.min() < 0 or tokens.max() >= L):
        raise IndexError("token id out of vocabulary range")
    return np.asarray(shard[tokens], dtype=np.float64)


def request_counts_columnwise(tokens, N):
    """Lookup requests served by each column shard: every shard serves every
    token ("each partition will get the same amount of requests")."""
    return [int(np.asarray(tokens).size)] * N


def request_counts_rowwise(tokens, L, N):
    """Lookup requests served by each row-wise shard (the imbalance argument
    of PAPER.md:272-273)."""
    tokens = np.asarray(tokens, dtype=np.int64)
    return [int(((tokens >= a) & (tokens < b)).sum()) for (a, b) in row_ranges(L, N)]


def request_counts_rowwise_hashed(tokens, N):
    """Row-wise partition with rows dealt round-robin (owner = id mod N), the
    usual fix for frequency-sorted vocabularies; still imbalanced when a few
    ids dominate."""
    tokens = np.asarray(tokens, dtype=np.int64)
    return [int((tokens % N == s).sum()) for s in range(N)]


def forward_bytes_out(ids_all, L, D, N, scheme, esz=4):
    """NVLink bytes each owner s SENDS in one forward exchange (the lookup
    results other ranks need), self-delivery excluded:
      column-wise  every owner sends every other rank's tokens, d = D/N columns:
                   (T - T_s) * (D/N) * e  (balanced);
      row / hash   owner s sends full rows for the tokens of other ranks that
                   fall in its rows: count_{r != s}(ids_r owned by s) * D * e."""
    T = [int(np.asarray(x).size) for x in ids_all]
    if scheme == "column":
        d = D // N
        return [(sum(T) - T[s]) * d * esz for s in range(N)]
    out = []
    for s in range(N):
        c = 0
        for r in range(N):
            if r == s:
                continue
            if scheme == "row":
                c += request_counts_rowwise(ids_all[r], L, N)[s]
            elif scheme == "hash":
                c += request_counts_rowwise_hashed(ids_all[r], N)[s]
            else:
                raise ValueError(scheme)
        out.append(c * D * esz)
    return out
