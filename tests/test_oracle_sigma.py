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
            # sigma_W (reading B12): |W| + |dW| + the first-order error of alpha m / (sqrt(v) + eps)
            # from the magnitudes summed into m and v, capped at twice Adam's largest possible step;
            # at the cancelled element (v = 0, denominator eps) it is the cap
            a1 = 1e-3 * np.sqrt(1 - B2) / (1 - B1)
            cap = 2 * a1 * (1 - B1) / np.sqrt((1 - B2) * (1 - B1 ** 2 / B2))
            sg = res.sigma_g
            mu_m = (1 - B1) * sg
            mu_v = (1 - B2) * (g * g + 2 * np.abs(g) * sg)
            sv = np.sqrt(v1)
            first = a1 * mu_m / (sv + 1e-8) + np.where(sv > 0, a1 * m1 * mu_v / (2 * np.where(sv > 0, sv, 1)
                                                                                   * (sv + 1e-8) ** 2), 0)
            want = np.abs(W[res.U]) + np.abs(dW) + np.minimum(cap, first)
            np.testing.assert_allclose(res.sigma_W, want, rtol=1e-12)
            assert res.sigma_W[0, 0] == pytest.approx(abs(W[5, 0]) + cap, rel=1e-12)


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
    # sigma_W >= |W_old| + |dW|, and never more than that plus twice Adam's largest step
    a1 = 1e-3 * np.sqrt(1 - B2) / (1 - B1)
    cap = 2 * a1 * (1 - B1) / np.sqrt((1 - B2) * (1 - B1 ** 2 / B2))
    base = np.abs(W[res.U]) + np.abs(dW)
    assert np.all(res.sigma_W >= base * (1 - 1e-12)) and np.all(res.sigma_W <= base + cap * (1 + 1e-12))


def _adam_fp32_like_gpu(w, m, v, g, alpha, b1=B1, b2=B2, eps=1e-8):
    """One Adam element step in fp32 with the GPU kernel's operation order
    (csrc/k_bwd.cu opt_math): m += (1-b1)(g-m); v += (1-b2)(g^2-v);
    w -= alpha * m * (1 / (sqrt(v) + eps)), every operation rounded to fp32."""
    f = np.float32
    w, m, v, g, alpha = f(w), f(m), f(v), f(g), f(alpha)
    m = f(m + f(f(1 - b1) * f(g - m)))
    v = f(v + f(f(1 - b2) * f(f(g * g) - v)))
    q = f(1) / f(f(np.sqrt(v)) + f(eps))
    return float(f(w - f(f(alpha * m) * q))), float(m), float(v)


def test_sigma_w_adam_covers_fp32_cancellation_in_m():
    """The Adam sigma_W term of reading B12 is NEEDED and SUFFICIENT: when g
    nearly cancels the previous m (m_new << |m_old|, |g|), an fp32 evaluation
    in the GPU's operation order misses the fp64 result by far more than
    1e-5 (|W_old| + |dW|), but stays within 1e-5 of the B12 sigma_W."""
    rng = np.random.default_rng(41)
    n = 4000
    m_old = rng.uniform(-0.05, 0.05, n).astype(np.float32).astype(np.float64)
    v_old = (m_old ** 2 * rng.uniform(1, 30, n)).astype(np.float32).astype(np.float64)
    g = (-B1 / (1 - B1) * m_old * (1 + rng.uniform(-1e-4, 1e-4, n))).astype(np.float32).astype(np.float64)
    W0 = rng.uniform(-1e-5, 1e-5, n).astype(np.float32).astype(np.float64)
    shards = [W0.reshape(n, 1).copy()]
    m, v = [m_old.reshape(n, 1).copy()], [v_old.reshape(n, 1).copy()]
    ids = [np.arange(n)]
    res = exchange.simulate_iteration(shards, ids, [g.reshape(n, 1)], None, 3, "coal", "fp64",
                                      exchange.OptimConfig("adam", lr=1e-3, grad_scale=1.0), m, v)
    a3 = 1e-3 * np.sqrt(1 - B2 ** 3) / (1 - B1 ** 3)
    gpu = np.array([_adam_fp32_like_gpu(W0[i], m_old[i], v_old[i], g[i], a3)[0] for i in range(n)])
    ref = shards[0][:, 0]
    err_new = np.abs(gpu - ref) / np.maximum(np.abs(ref), res.sigma_W[:, 0])
    err_old = np.abs(gpu - ref) / np.maximum(np.abs(ref), np.abs(W0) + np.abs(ref - W0))
    assert err_new.max() <= 1e-5
    assert err_old.max() > 1e-5


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
