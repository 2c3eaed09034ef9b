"""Pins for the oracle's tolerance normalisers (SURVEY §8(c) "Comparison
metric"): sigma_g = scale * sum of |terms| of every merged
gradient element, sigma_W / sigma_m / sigma_v = the first-order magnitudes of
the updated W, m, v.  Every float tolerance of the GPU parity tests divides by
them, so they are pinned here to exact values — by brute force over integer
gradients (sums of small integers are exact in fp64) and by a hand-computed
cancellation case — and the bound they define is checked against the actual
rounding error of fp32 summation in arbitrary order."""

import numpy as np
import pytest

from oracle import exchange, partition

B1, B2 = 0.9, 0.999


def _brute_sigma_g(L, D, ids, dY, scale, pad_id=-1):
    """scale * sum over every (rank, position) holding id u of |dY[j, c]| —
    a plain double loop, independent of the oracle's coalesce."""
    S = np.zeros((L, D))
    G = np.zeros((L, D))
    for r in range(len(ids)):
        for j, u in enumerate(ids[r]):
            if pad_id >= 0 and u == pad_id:
                continue
            for c in range(D):
                S[u, c] += abs(float(dY[r][j][c]))
                G[u, c] += float(dY[r][j][c])
    return scale * S, scale * G


@pytest.mark.parametrize("N", [1, 2, 4])
@pytest.mark.parametrize("mode", ["raw", "coal", "split"])
def test_sigma_g_brute_force_integer_gradients(N, mode):
    rng = np.random.default_rng(11 + N)
    L, D = 40, 8
    ids = [rng.integers(0, L, size=rng.integers(5, 30)) for _ in range(N)]
    dY = [rng.integers(-9, 10, size=(len(x), D)).astype(np.float64) for x in ids]
    nxt = [rng.integers(0, L, size=10) for _ in range(N)]
    W = rng.integers(-5, 6, size=(L, D)).astype(np.float64)
    shards = partition.partition_columnwise(W, N)
    res = exchange.simulate_iteration(shards, ids, dY, nxt, 1, mode, "fp64",
                                      exchange.OptimConfig("sgd", lr=0.25))
    S, G = _brute_sigma_g(L, D, ids, dY, 1.0 / N)
    np.testing.assert_array_equal(res.sigma_g, S[res.U])
    np.testing.assert_array_equal(res.g, G[res.U])
    # SGD: sigma_W = |W_old| + lr * sigma_g, exactly
    np.testing.assert_array_equal(res.sigma_W, np.abs(W[res.U]) + 0.25 * S[res.U])


def test_sigma_hand_computed_cancellation():
    """Two ranks, id 5 gets +3 and -3 in column 0 (g = 0, sigma_g = 3), +1 and
    +2 in column 1.  Column 0 is the case the normaliser exists for: |ref| = 0
    after cancellation, so plain relative error is undefined and the sigma
    metric falls back to the magnitude of what was summed."""
    ids = [np.array([5, 7]), np.array([5])]
    dY = [np.array([[3.0, 1.0], [1.0, 1.0]]), np.array([[-3.0, 2.0]])]
    W = np.zeros((8, 2))
    W[5] = [0.5, -0.25]
    W[7] = [-1.0, 2.0]
    for kind in ("sgd", "adam"):
        shards = partition.partition_columnwise(W.copy(), 1)
        m = [np.zeros_like(shards[0])] if kind == "adam" else None
        v = [np.zeros_like(shards[0])] if kind == "adam" else None
        lr = 0.1 if kind == "sgd" else 1e-3
        res = exchange.simulate_iteration(shards, [np.concatenate(ids)], [np.vstack(dY)], None, 1, "coal", "fp64",
                                          exchange.OptimConfig(kind, lr=lr, grad_scale=0.5), m, v)
        assert res.U.tolist() == [5, 7]
        np.testing.assert_array_equal(res.g, [[0.0, 1.5], [0.5, 0.5]])
        np.testing.assert_array_equal(res.sigma_g, [[3.0, 1.5], [0.5, 0.5]])
        if kind == "sgd":
            np.testing.assert_allclose(res.sigma_W, [[0.5 + 0.3, 0.25 + 0.15], [1.0 + 0.05, 2.0 + 0.05]],
                                       rtol=1e-15)
        else:
            g = res.g
            # step 1 from m = v = 0: m = (1-b1) g, v = (1-b2) g^2, stored fp32 (reading R11)
            m1 = np.abs((((1 - B1) * g).astype(np.float32)).astype(np.float64))
            v1 = ((1 - B2) * g * g).astype(np.float32).astype(np.float64)
            np.testing.assert_allclose(res.sigma_m, m1 + (1 - B1) * res.sigma_g, rtol=1e-15)
            np.testing.assert_allclose(res.sigma_v, v1 + 2 * (1 - B2) * np.abs(g) * res.sigma_g, rtol=1e-15)
            # the cancelled element: g = 0 -> m = v = 0, W unchanged, sigma_m = (1-b1) * 3
            assert res.sigma_m[0, 0] == pytest.approx((1 - B1) * 3.0, rel=1e-15)
            assert res.sigma_v[0, 0] == 0.0
            dW = shards[0][res.U] - W[res.U]
            assert dW[0, 0] == 0.0
            np.testing.assert_allclose(res.sigma_W, np.abs(W[res.U]) + np.abs(dW), rtol=1e-15)


def test_sigma_bounds_fp32_summation_error():
    """The metric's premise: an fp32 sum of the same terms in ANY order differs
    from the exact sum by at most gamma_{n-1} * sum|terms| (Higham) — i.e. by
    a small multiple of u * sigma_g, far inside 1e-5 * sigma_g — while a
    dropped or sign-flipped term (a plausible bug) moves the sum by one term,
    far outside it.  Checked on Zipf-head-like segments with cancellation."""
    rng = np.random.default_rng(5)
    u32 = 2.0 ** -24
    for n in (2, 17, 1000, 5000):
        terms = rng.uniform(-1, 1, n).astype(np.float32).astype(np.float64)
        exact = float(np.sum(terms, dtype=np.float64))
        sigma = float(np.abs(terms).sum())
        gamma = (n - 1) * u32 / (1 - (n - 1) * u32)
        for _ in range(5):
            perm = rng.permutation(n)
            acc = np.float32(0.0)
            for x in terms[perm].astype(np.float32):
                acc = np.float32(acc + x)
            err = abs(float(acc) - exact)
            assert err <= gamma * sigma
            assert err / max(abs(exact), sigma) <= 1e-5 or n * u32 > 1e-5
        # a dropped term is detected
        k = int(np.argmax(np.abs(terms)))
        bad = exact - terms[k]
        assert abs(bad - exact) / max(abs(exact), sigma) > 1e-5


def test_sigma_adam_closed_form_step1():
    """Adam step 1 from m = v = 0 (SURVEY §8(c) pins): dW = -lr g / (|g| + eps/sqrt(1-b2));
    sigma_W = |W_old| + |dW| exactly that."""
    rng = np.random.default_rng(3)
    L, D = 20, 4
    ids = [rng.integers(0, L, 12)]
    dY = [rng.uniform(-1, 1, (12, D))]
    W = rng.uniform(-0.05, 0.05, (L, D))
    shards = partition.partition_columnwise(W.copy(), 1)
    m, v = [np.zeros((L, D))], [np.zeros((L, D))]
    res = exchange.simulate_iteration(shards, ids, dY, None, 1, "split", "fp64",
                                      exchange.OptimConfig("adam", lr=1e-3, grad_scale=1.0), m, v)
    g = res.g
    dW = -1e-3 * g / (np.abs(g) + 1e-8 / np.sqrt(1 - B2))
    np.testing.assert_allclose(shards[0][res.U] - W[res.U], dW, rtol=1e-9, atol=1e-18)
    np.testing.assert_allclose(res.sigma_W, np.abs(W[res.U]) + np.abs(dW), rtol=1e-9)


def test_metric_helpers():
    """tests/_metric.py: the accumulated-sigma store and the bf16 update bound."""
    from _metric import SigmaAcc, assert_close_acc, assert_update, ulp_bf16
    a = SigmaAcc(2)
    a.add(np.array([3, 7]), np.array([[1.0, 2.0], [3.0, 4.0]]))
    a.add(np.array([1, 7]), np.array([[5.0, 5.0], [1.0, 1.0]]))
    np.testing.assert_array_equal(a.ids, [1, 3, 7])
    np.testing.assert_array_equal(a.get(np.array([7, 2, 1, 7])), [[4, 5], [0, 0], [5, 5], [4, 5]])
    s = a.snapshot()
    a.add(np.array([2]), np.ones((1, 2)))
    assert s.ids.tolist() == [1, 3, 7]
    # untouched values must be equal exactly; touched ones within tol * sigma
    assert_close_acc(np.array([1.0, 2.0 + 1e-6]), np.array([1.0, 2.0]), np.array([0.0, 1.0]), "fp32") < 1e-5 + 1e-12
    with pytest.raises(AssertionError):
        assert_close_acc(np.array([1.0 + 1e-12]), np.array([1.0]), np.array([0.0]), "fp32")
    # bf16 ulp: 2^-7 relative at the bottom of each binade
    assert ulp_bf16(1.0) == 2.0 ** -7 and ulp_bf16(0.03) == 2.0 ** -6 * 2.0 ** -7
    # an update off by 50 % fails, one ulp passes
    old, ref = np.array([0.03]), np.array([0.03 - 1e-3])
    assert_update(ref + ulp_bf16(ref), ref, old)
    with pytest.raises(AssertionError):
        assert_update(old - 0.5e-3, ref, old)
