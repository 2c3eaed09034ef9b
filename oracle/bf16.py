"""Storage / wire rounding points (oracle; test infrastructure only).

The paper never states its precision ("each taking over 1.5GB"
implies fp32 for LM; reading R11 fixes bf16 storage + wire for the
other configs, fp32 accumulation).  These functions are the *definitions* of
round-to-nearest-even onto the fp32 and bf16 grids, written from the IEEE-754
definition (significand of p bits, ties to even), not from bit tricks.
"""

import numpy as np

# p = number of significand bits including the implicit one.
_P = {"fp32": 24, "bf16": 8}
# largest finite value of each format: (2 - 2^(1-p)) * 2^emax, emax = 127 for both
_EMAX = 127
_EMIN = -126


def round_to(x, dtype):
    """Round fp64 values to the nearest value of ``dtype`` ("fp32"/"bf16"/"fp64"),
    ties to even, returned as fp64 (so it can keep flowing through fp64 math).

    Definition: write |x| = f * 2^e with f in [1, 2); the representable
    neighbours are multiples of 2^(e - (p-1)) (for e below emin the spacing
    stays 2^(emin - (p-1)) — subnormals).  np.rint rounds half to even.
    Overflow past the largest finite value goes to +-inf.
    """
    x = np.asarray(x, dtype=np.float64)
    if dtype == "fp64":
        return x.copy()
    p = _P[dtype]
    out = np.zeros_like(x)
    nz = (x != 0) & np.isfinite(x)
    ax = np.abs(x[nz])
    # frexp: ax = m * 2^k, m in [0.5, 1)  ->  ax = (2m) * 2^(k-1), 2m in [1, 2)
    _, k = np.frexp(ax)
    e = np.maximum(k - 1, _EMIN)
    ulp = np.ldexp(1.0, e - (p - 1))
    r = np.rint(ax / ulp) * ulp
    maxfin = (2.0 - 2.0 ** (1 - p)) * 2.0 ** _EMAX
    r = np.where(r > maxfin, np.inf, r)
    out[nz] = np.sign(x[nz]) * r
    out[~np.isfinite(x)] = x[~np.isfinite(x)]
    return out


def is_representable(x, dtype):
    """True where x already lies on the ``dtype`` grid."""
    x = np.asarray(x, dtype=np.float64)
    return round_to(x, dtype) == x
