"""Collective primitives over N simulated workers (oracle; test infrastructure only).

PAPER.md:94-106 (§2.1) and Fig. 1:
  * AllReduce "aggregates data from all processes, reduces the data with an
    operator such as sum, and distributes results back";
  * AllGather "gathers the complete data from all tasks and distributes the
    combined data to all tasks";
  * AlltoAll "redistribute[s] the data among all processes where processes
    transmit and receive data from every other process" —
    a block transpose: rank s's output slot r = rank r's input block s.

A "group" is just a Python list indexed by rank.  Sums run in ascending rank
order (deterministic), fp64.
"""

import numpy as np


def all_reduce(xs):
    """Every rank gets sum_r xs[r] (rank-ascending fp64 sum)."""
    acc = np.zeros_like(np.asarray(xs[0], dtype=np.float64))
    for x in xs:
        acc = acc + np.asarray(x, dtype=np.float64)
    return [acc.copy() for _ in xs]


def all_gather(payloads):
    """Every rank gets [payload_0, ..., payload_{N-1}] (indexed by source)."""
    return [[p for p in payloads] for _ in payloads]


def all_to_all(blocks):
    """blocks[r][s] = block rank r sends to rank s.  Returns out with
    out[s][r] = blocks[r][s] (block transpose)."""
    N = len(blocks)
    for r in range(N):
        if len(blocks[r]) != N:
            raise ValueError("collective-contract error: wrong block count")
    return [[blocks[r][s] for r in range(N)] for s in range(N)]


def alltoall_sent_elems(blocks):
    """Elements each rank actually transmits, self-delivery excluded
    (SPEC.md:227 measure_bytes)."""
    N = len(blocks)
    return [sum(int(np.asarray(blocks[r][s]).size) for s in range(N) if s != r) for r in range(N)]


def allgather_sent_elems(payloads):
    """AllGather: each rank sends its payload to the N-1 others."""
    N = len(payloads)
    return [(N - 1) * int(np.asarray(p).size) for p in payloads]
