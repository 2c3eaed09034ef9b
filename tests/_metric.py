"""Comparison metric of SURVEY §8(c):

  integers: equal exactly;  forward Y: equal exactly (pure copies);
  reduced floats: err_i = |gpu_i - ref_i| / max(|ref_i|, sigma_i) <= tol,
  tol = 1e-5 (fp32) / 2e-2 (bf16) (BASELINE.json north_star),
  sigma_i = first-order magnitude the oracle computes next to each value.
"""

import numpy as np

TOL = {"fp32": 1e-5, "bf16": 2e-2}


def sigma_err(gpu, ref, sigma):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.maximum(np.abs(ref), np.asarray(sigma, np.float64))
    den = np.where(den == 0, 1.0, den)
    return np.abs(gpu - ref) / den


def assert_close(gpu, ref, sigma, dtype, what=""):
    e = sigma_err(gpu, ref, sigma)
    if e.size == 0:
        return 0.0
    worst = float(e.max())
    if not worst <= TOL[dtype]:
        i = np.unravel_index(int(np.argmax(e)), e.shape)
        raise AssertionError(f"{what}: max sigma-normalised error {worst:.3e} > {TOL[dtype]} at {i}: "
                             f"gpu={np.asarray(gpu)[i]!r} ref={np.asarray(ref)[i]!r} sigma={np.asarray(sigma)[i]!r}")
    return worst
