"""B200-native EmbRace sparse-embedding exchange (arXiv 2110.09132).

The product is libembrace.so (C ABI, include/embrace.h) built from csrc/ for
sm_100a; ``embrace`` is its thin ctypes binding and ``runtime`` the
process-group bootstrap.  There is no CPU fallback.
"""

from . import embrace  # noqa: F401
