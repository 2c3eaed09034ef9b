"""Comparison metric of SURVEY §8(c) (DESIGN.md §11 "Parity"):

  integers: equal exactly;  forward Y: equal exactly (pure copies);
  reduced floats: err_i = |gpu_i - ref_i| / max(|ref_i|, sigma_i) <= tol,
  tol = 1e-5 (fp32) / 2e-2 (bf16) (BASELINE.json north_star),
  sigma_i = first-order magnitude the oracle computes next to each value.

Free-running comparisons (no resync of the oracle to the GPU state) use the
same bound with sigma accumulated over the iterations that touched a row
(SigmaAcc): every step adds at most tol * sigma_k of rounding difference
(per-step bound above), SGD propagates an earlier difference unchanged and
Adam's moments damp theirs (beta < 1), so after K steps the difference is at
most tol * sum_k sigma_k.

bf16 updates are also checked against the SIZE of the update: one Adam step
(~lr = 1e-3) is far below sigma_W ~ |W| ~ 0.03, so the sigma metric alone
would pass an update wrong by ~50 %.  assert_update requires
|gpu - ref| <= ulp_bf16(ref) + 2e-2 * |ref - W_old|: one ulp for the RNE
straddle of fp32 vs fp64 math, 2 % of the update for the sender-side bf16
wire rounding of the coalesced gradient (<= 2^-8 relative per source).
"""

import numpy as np

TOL = {"fp32": 1e-5, "bf16": 2e-2}
UPDATE_REL = 2e-2


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


def assert_close_acc(gpu, ref, sigma_acc, dtype, what=""):
    """Free-running bound: |gpu - ref| <= tol * max(|ref|, sigma_acc); where
    sigma_acc == 0 (a value no update has touched) the values must be equal."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    sig = np.asarray(sigma_acc, np.float64)
    untouched = sig == 0
    if np.any(untouched) and not np.array_equal(gpu[untouched], ref[untouched]):
        i = np.argwhere(untouched & (gpu != ref))[0]
        raise AssertionError(f"{what}: untouched value differs at {tuple(i)}: gpu={gpu[tuple(i)]!r} "
                             f"ref={ref[tuple(i)]!r}")
    return assert_close(gpu, ref, np.where(untouched, 0.0, sig), dtype, what)


def ulp_bf16(x):
    """Spacing of the bf16 grid at |x| (8 significand bits; normal range)."""
    ax = np.abs(np.asarray(x, np.float64))
    _, e = np.frexp(np.where(ax == 0, 2.0 ** -126, ax))     # ax = f * 2^e, f in [0.5, 1)
    return np.ldexp(1.0, np.maximum(e - 1, -126) - 7)


def assert_update(gpu, ref, old, what=""):
    """bf16 rows after one update: |gpu - ref| <= ulp(ref) + 2e-2 |ref - old|.
    Returns the worst |gpu - ref| / (ulp(ref) + 2e-2 |ref - old|)."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    old = np.asarray(old, np.float64)
    if gpu.size == 0:
        return 0.0
    bound = ulp_bf16(ref) + UPDATE_REL * np.abs(ref - old)
    e = np.abs(gpu - ref) / bound
    worst = float(e.max())
    if not worst <= 1.0:
        i = np.unravel_index(int(np.argmax(e)), e.shape)
        raise AssertionError(f"{what}: |gpu - ref| = {abs(gpu[i] - ref[i]):.3e} > ulp + 2% of the update "
                             f"({bound[i]:.3e}) at {i}: gpu={gpu[i]!r} ref={ref[i]!r} old={old[i]!r}")
    return worst


class SigmaAcc:
    """Per-row sigma accumulated over iterations: rows (ascending int64 ids) and
    an fp64 [rows, D] sum of the per-iteration sigma of those rows."""

    def __init__(self, D):
        self.D = D
        self.ids = np.zeros(0, np.int64)
        self.val = np.zeros((0, D))

    def add(self, rows, sigma):
        rows = np.asarray(rows, np.int64)
        allids = np.union1d(self.ids, rows)
        new = np.zeros((allids.size, self.D))
        new[np.searchsorted(allids, self.ids)] = self.val
        new[np.searchsorted(allids, rows)] += np.asarray(sigma, np.float64)
        self.ids, self.val = allids, new

    def get(self, rows):
        """sigma rows for ids `rows` (any order, repeats allowed); 0 where never added."""
        rows = np.asarray(rows, np.int64)
        out = np.zeros((rows.size, self.D))
        if self.ids.size:
            pos = np.searchsorted(self.ids, rows).clip(0, self.ids.size - 1)
            hit = self.ids[pos] == rows
            out[hit] = self.val[pos[hit]]
        return out

    def snapshot(self):
        s = SigmaAcc(self.D)
        s.ids, s.val = self.ids.copy(), self.val.copy()
        return s
