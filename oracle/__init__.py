"""EmbRace CPU oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct NumPy (fp64) statement of what the
paper's Sparsity-aware Hybrid Communication hot path computes
(arXiv 2110.09132, /root/reference/PAPER.md).  Every function cites the
PAPER.md line (and section / table / algorithm) it restates.

Rules this package follows:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import it.  The product
    (``paper_2110_09132_b200``) never imports it and never falls back to it.
  * It shares no code with the CUDA path (no common helpers, tables or
    constants).  Both sides are fed by ``synthetic/`` (seeded input
    generators, no method arithmetic).
  * Math is fp64.  The only rounding points are the ones the method has on a
    real machine: table storage (fp32 / bf16), the wire dtype of coalesced
    gradients, and fp32 storage of Adam moments (readings R11).
  * Library primitives (stable sort, np.unique, np.add.reduceat) serve as
    single steps; there is no blocking, fusion or reordering beyond the
    paper's own statement.

Parity pins: every function is pinned by ``tests/test_oracle_*.py`` against
worked examples (tests/golden/, each cited), closed forms, invariants or
brute force.  Throughput is "parity unpinned" (the paper prints no number
for this path).
"""

from . import bf16, collectives, cost, exchange, optim, partition, schedule, sparse  # noqa: F401
