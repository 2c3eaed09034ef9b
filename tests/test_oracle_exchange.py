"""Pins for the oracle's simulated N-worker exchange: the plain definition
(dense lookup / dense scatter-add / one optimizer step, brute force on tiny
vocabularies), the paper's invariants, and the byte closed forms."""

import json
import os

import numpy as np
import pytest

from oracle import bf16, cost, exchange, optim, partition
from synthetic import get_config, make_workload
from synthetic.workloads import Config, gen_table

SGD = exchange.OptimConfig("sgd", lr=0.1)
ADAM = exchange.OptimConfig("adam", lr=1e-3)


def _tiny(N, iters=3, cfg=None):
    cfg = cfg or get_config("tiny")
    return cfg, make_workload(cfg, N, iters), gen_table(cfg).astype(np.float64)


def _brute_dense_sgd(W, ids, dY, lr, scale, pad_id=-1):
    """Independent brute force: dense L x D gradient by triple loop, dense step."""
    G = np.zeros_like(W)
    hit = np.zeros(W.shape[0], bool)
    for r in range(len(ids)):
        for j in range(len(ids[r])):
            u = int(ids[r][j])
            if pad_id >= 0 and u == pad_id:
                continue
            for c in range(W.shape[1]):
                G[u, c] += float(dY[r][j][c])
            hit[u] = True
    return W - lr * scale * G, hit


@pytest.mark.parametrize("N", [1, 2, 4])
@pytest.mark.parametrize("mode", ["raw", "coal", "split"])
def test_sgd_exchange_equals_dense_sgd_step(N, mode):
    cfg, wl, W = _tiny(N)
    shards = partition.partition_columnwise(W, N)
    res = exchange.simulate_iteration(shards, wl.ids[0], wl.dY[0], wl.ids[1], 1, mode, "fp64", SGD)
    ref, hit = _brute_dense_sgd(W, wl.ids[0], wl.dY[0], 0.1, 1.0 / N)
    np.testing.assert_allclose(np.hstack(shards), ref, rtol=0, atol=1e-13)
    # forward: hconcat of shard lookups == dense lookup, bit-exact
    for s in range(N):
        np.testing.assert_array_equal(res.Y[s], W[wl.ids[0][s]])
    assert res.U.tolist() == np.flatnonzero(hit).tolist()


def test_sgd_pad_rows_dropped_when_pad_id_set():
    cfg, wl, W = _tiny(2)
    shards = partition.partition_columnwise(W, 2)
    exchange.simulate_iteration(shards, wl.ids[0], wl.dY[0], wl.ids[1], 1, "split", "fp64", SGD, pad_id=0)
    ref, _ = _brute_dense_sgd(W, wl.ids[0], wl.dY[0], 0.1, 0.5, pad_id=0)
    new = np.hstack(shards)
    np.testing.assert_allclose(new, ref, rtol=0, atol=1e-13)
    assert np.array_equal(new[0], W[0])   # pad row untouched


def test_adam_exchange_equals_dense_reference_multi_step():
    N = 2
    cfg, wl, W = _tiny(N, iters=4)
    shards = partition.partition_columnwise(W, N)
    m = [np.zeros_like(s) for s in shards]
    v = [np.zeros_like(s) for s in shards]
    Wd, md, vd = W.copy(), np.zeros_like(W), np.zeros_like(W)
    for t in range(1, 4):
        exchange.simulate_iteration(shards, wl.ids[t - 1], wl.dY[t - 1], wl.ids[t], t, "split", "fp64",
                                    ADAM, m, v)
        exchange.dense_reference(Wd, wl.ids[t - 1], wl.dY[t - 1], t, "fp64", ADAM, md, vd)
        # m, v are stored fp32 in both (rounding point of the GPU's storage)
    np.testing.assert_allclose(np.hstack(shards), Wd, rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.hstack(m), md, rtol=0, atol=1e-12)


@pytest.mark.parametrize("dtype", ["fp64", "fp32", "bf16"])
@pytest.mark.parametrize("kind", ["sgd", "adam"])
def test_split_equals_coal_bitwise(dtype, kind):
    """Two disjoint parts with the same per-row arithmetic == one part."""
    N = 4
    cfg, wl, W = _tiny(N)
    W = bf16.round_to(W, dtype) if dtype != "fp64" else W
    dY = [[bf16.round_to(x, dtype) for x in it] for it in wl.dY]
    opt = SGD if kind == "sgd" else ADAM
    out = {}
    for mode in ("coal", "split"):
        shards = partition.partition_columnwise(W, N)
        m = [np.zeros_like(s) for s in shards]
        v = [np.zeros_like(s) for s in shards]
        for t in (1, 2):
            exchange.simulate_iteration(shards, wl.ids[t - 1], dY[t - 1], wl.ids[t], t, mode, dtype, opt, m, v)
        out[mode] = (np.hstack(shards), np.hstack(m), np.hstack(v))
    for a, b in zip(out["coal"], out["split"]):
        assert np.array_equal(a, b)


def test_raw_vs_coal_differ_only_by_wire_rounding():
    N = 2
    cfg, wl, W = _tiny(N)
    res = {}
    for mode in ("raw", "coal"):
        shards = partition.partition_columnwise(W, N)
        res[mode] = exchange.simulate_iteration(shards, wl.ids[0], wl.dY[0], wl.ids[1], 1, mode, "fp64", SGD)
    np.testing.assert_array_equal(res["raw"].U, res["coal"].U)
    np.testing.assert_allclose(res["raw"].g, res["coal"].g, rtol=1e-14, atol=1e-15)


def test_invariants_and_byte_closed_forms():
    for N in (1, 2, 4):
        cfg, wl, W = _tiny(N)
        shards = partition.partition_columnwise(W, N)
        res = exchange.simulate_iteration(shards, wl.ids[0], wl.dY[0], wl.ids[1], 1, "split", "fp32", SGD)
        nxt = set(np.concatenate(wl.ids[1]).tolist())
        assert set(res.P) | set(res.Q) == set(res.U) and not (set(res.P) & set(res.Q))
        assert set(res.P) <= nxt
        assert all(res.p[n] <= res.u[n] <= res.T[n] for n in range(N))
        d, e = cfg.D // N, 4
        # every shard serves exactly T lookups
        for r in range(N):
            assert res.fwd_bytes[r].sum() == res.T.sum() * d * e
        # uniform case: one AlltoAll of total payload aM = T_r*D elems sends (N-1) aM / N
        if len(set(res.T.tolist())) == 1:
            aM = int(res.T[0]) * cfg.D
            assert res.sent("fwd")[0] == cost.alltoall_bandwidth_numerator(N, aM) * e
        for n in range(N):
            assert res.sent("bwd")[n] == (N - 1) * res.u[n] * d * e
            assert res.sent("ids")[n] == (N - 1) * res.T[n] * 4
        if N == 1:
            assert res.sent("fwd")[0] == res.sent("bwd")[0] == res.sent("ids")[0] == 0


def test_prior_part_guarantee():
    """After only the prior part is applied, every row the next batch reads
    already holds its fully-updated value."""
    N = 2
    cfg, wl, W = _tiny(N)
    full = partition.partition_columnwise(W, N)
    res = exchange.simulate_iteration(full, wl.ids[0], wl.dY[0], wl.ids[1], 1, "split", "fp64", SGD)
    prior_only = np.array(W, copy=True)
    at = np.searchsorted(res.U, res.P)
    optim.sgd_apply(prior_only, res.P, res.g[at], 0.1)
    nxt = np.unique(np.concatenate(wl.ids[1]))
    np.testing.assert_array_equal(prior_only[nxt], np.hstack(full)[nxt])


def test_last_step_everything_scheduled():
    cfg, wl, W = _tiny(2)
    shards = partition.partition_columnwise(W, 2)
    res = exchange.simulate_iteration(shards, wl.ids[0], wl.dY[0], None, 1, "split", "fp64", SGD)
    assert res.P.size == 0 and res.Q.tolist() == res.U.tolist()


def test_empty_rank_batch():
    cfg, wl, W = _tiny(2)
    ids = [wl.ids[0][0], np.zeros(0, np.int32)]
    dY = [wl.dY[0][0], np.zeros((0, cfg.D), np.float32)]
    shards = partition.partition_columnwise(W, 2)
    res = exchange.simulate_iteration(shards, ids, dY, wl.ids[1], 1, "split", "fp64", SGD)
    assert res.Y[1].shape == (0, cfg.D) and res.u[1] == 0
    ref, _ = _brute_dense_sgd(W, ids, dY, 0.1, 0.5)
    np.testing.assert_allclose(np.hstack(shards), ref, atol=1e-13, rtol=0)


def test_out_of_range_id_rejected():
    cfg, wl, W = _tiny(2)
    ids = [np.array([0, 1000]), wl.ids[0][1]]
    with pytest.raises(IndexError):
        exchange.simulate_iteration(partition.partition_columnwise(W, 2), ids, wl.dY[0], None, 1)


def test_bf16_wire_rounding_point():
    """COAL/SPLIT in bf16 send round_bf16(sum) — RAW sums the raw bf16 slices."""
    N = 2
    cfg, wl, W = _tiny(N)
    W = bf16.round_to(W, "bf16")
    dY = [bf16.round_to(x, "bf16") for x in wl.dY[0]]
    r = {}
    for mode in ("raw", "coal"):
        r[mode] = exchange.simulate_iteration(partition.partition_columnwise(W, N), wl.ids[0], dY, wl.ids[1],
                                              1, mode, "bf16", SGD)
    # COAL merged gradient = scale * sum_n round_bf16(Gc_n); RAW = scale * sum_n Gc_n
    diff = np.abs(r["raw"].g - r["coal"].g)
    assert diff.max() > 0                       # the rounding point is real
    assert np.all(diff <= 2 ** -8 * r["raw"].sigma_g + 1e-30)   # <= one bf16 half-ulp per source


def test_paper_table_arithmetic():
    """Config shapes and the §4.2.2 percentages agree with PAPER.md's tables."""
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables.json")))
    lm = get_config("lstm_lm")
    assert round(2 * lm.L * lm.D / 1e6, 2) == gold["table1_embedding_params_M"]["LM"]
    assert round(2 * 32_317 * 1024 / 1e6, 2) == gold["table1_embedding_params_M"]["GNMT-8"]
    assert round(30_528 * 768 / 1e6, 2) == gold["table1_embedding_params_M"]["BERT-base"]
    for k, (orig, coal, prior) in ((k, x) for k, x in gold["table3_rows"].items() if k != "cite"):
        # the text's percentages agree with Table 3 to 0.1 points (GNMT: 53.16 printed 53.1)
        assert abs(100 * (1 - coal / orig) - gold["coalesce_reduction_pct"][k]) <= 0.1
        assert abs(100 * (1 - prior / coal) - gold["prior_reduction_pct"][k]) <= 0.1


def test_oracle_lm_sized_sample_runs():
    """The LM-shaped workload runs through the oracle (N=1, one iteration)."""
    cfg = get_config("lstm_lm")
    small = Config("lm_slice", cfg.L, 32, "fp32", 128, 35, 18)   # narrow D keeps it fast
    wl = make_workload(small, 1, 2)
    W = gen_table(small)
    m, v = [np.zeros_like(W)], [np.zeros_like(W)]
    res = exchange.simulate_iteration([W], wl.ids[0], wl.dY[0], wl.ids[1], 1, "split", "fp32", ADAM, m, v)
    assert res.u[0] < res.T[0] and 0 < res.p[0] < res.u[0]


# ---------------------------------------------------------------- NEXT-3: several tables in one exchange

@pytest.mark.parametrize("mode", ["raw", "split"])
def test_stacked_tables_equal_separate_exchanges(mode):
    """Reading for SURVEY §8(f) NEXT-3 (PAPER.md:481 two LM tables; PAPER.md:319-320
    GNMT encoder / decoder tables): tables of one width stacked row-wise form ONE
    exchange over global row ids (local id + table base).  Pinned here: that
    exchange gives every table exactly what its own exchange gives (the row sets
    are disjoint, so sums, splits and updates are per table)."""
    rng = np.random.default_rng(31)
    L1, L2, D, N = 50, 30, 8, 2
    A = rng.uniform(-1, 1, (L1, D))
    B = rng.uniform(-1, 1, (L2, D))
    ia = [rng.integers(0, L1, 12) for _ in range(N)]
    ib = [rng.integers(0, L2, 7) for _ in range(N)]
    ga = [rng.uniform(-1, 1, (12, D)) for _ in range(N)]
    gb = [rng.uniform(-1, 1, (7, D)) for _ in range(N)]
    na = [rng.integers(0, L1, 5) for _ in range(N)]
    nb_ = [rng.integers(0, L2, 5) for _ in range(N)]
    # stacked: one exchange, global ids (B's rows after A's)
    S = partition.partition_columnwise(np.vstack([A, B]), N)
    ids = [np.concatenate([ia[r], L1 + ib[r]]) for r in range(N)]
    dY = [np.vstack([ga[r], gb[r]]) for r in range(N)]
    nxt = [np.concatenate([na[r], L1 + nb_[r]]) for r in range(N)]
    res = exchange.simulate_iteration(S, ids, dY, nxt, 1, mode, "fp64", SGD)
    # separate exchanges
    SA = partition.partition_columnwise(A.copy(), N)
    SB = partition.partition_columnwise(B.copy(), N)
    ra = exchange.simulate_iteration(SA, ia, ga, na, 1, mode, "fp64", SGD)
    rb = exchange.simulate_iteration(SB, ib, gb, nb_, 1, mode, "fp64", SGD)
    for r in range(N):
        np.testing.assert_array_equal(res.Y[r][:12], ra.Y[r])
        np.testing.assert_array_equal(res.Y[r][12:], rb.Y[r])
    np.testing.assert_array_equal(np.hstack(S)[:L1], np.hstack(SA))
    np.testing.assert_array_equal(np.hstack(S)[L1:], np.hstack(SB))
    assert res.U.tolist() == ra.U.tolist() + (L1 + rb.U).tolist()
