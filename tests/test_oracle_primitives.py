"""Pins for the oracle's primitives against worked examples, closed forms,
library routines and brute force (none of them re-types the oracle formula).
"""

import json
import os
import random

import numpy as np
import pytest

from oracle import bf16, collectives, cost, optim, partition, schedule, sparse

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


# ---------------------------------------------------------------- rounding
def test_round_fp32_matches_numpy_cast():
    # special case that reduces to a library routine: IEEE fp64 -> fp32 RNE
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.standard_normal(20000) * 10.0 ** rng.integers(-30, 30, 20000),
                        [0.0, -0.0, 1e-45, 3.4e38, -3.4e38, 1.5e-40]])
    np.testing.assert_array_equal(bf16.round_to(x, "fp32"), x.astype(np.float32).astype(np.float64))


def test_round_bf16_matches_torch_on_fp32_inputs():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(2)
    x = (rng.standard_normal(50000) * 10.0 ** rng.integers(-20, 20, 50000)).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(bf16.round_to(x.astype(np.float64), "bf16"), ref)


def test_round_bf16_ties_to_even_hand_values():
    # bf16 spacing at 1.0 is 2^-7; 1 + 2^-8 is a tie -> even (1.0);
    # 1 + 3*2^-8 is a tie between 1+2^-7 and 1+2^-6 -> even mantissa (1+2^-6)
    x = np.array([1 + 2.0 ** -8, 1 + 3 * 2.0 ** -8, -(1 + 2.0 ** -8), 1 + 2.0 ** -8 + 2.0 ** -20])
    np.testing.assert_array_equal(bf16.round_to(x, "bf16"), [1.0, 1 + 2.0 ** -6, -1.0, 1 + 2.0 ** -7])


# ---------------------------------------------------------------- sparse
def test_coalesce_worked_example():
    g = GOLD["coalesce"]
    ui, uv, _ = sparse.coalesce(g["idx"], g["val"])
    assert ui.tolist() == g["out_idx"]
    assert uv.tolist() == g["out_val"]


def test_coalesce_empty():
    ui, uv, _ = sparse.coalesce(np.zeros(0, np.int64), np.zeros((0, 3)))
    assert ui.size == 0 and uv.shape == (0, 3)


def _dict_coalesce(idx, val):
    """Independent brute force: Python dict accumulation."""
    acc = {}
    for i, row in zip(idx, val):
        acc.setdefault(int(i), np.zeros(len(row)))
        acc[int(i)] = acc[int(i)] + np.asarray(row, np.float64)
    ks = sorted(acc)
    return ks, [acc[k] for k in ks]


def test_coalesce_brute_force_and_invariants():
    rng = np.random.default_rng(3)
    for _ in range(300):
        c = int(rng.integers(0, 40))
        idx = rng.integers(0, 12, c)
        val = rng.integers(-5, 6, (c, 3)).astype(np.float64)   # integers: sums exact
        ui, uv, _ = sparse.coalesce(idx, val)
        ks, vs = _dict_coalesce(idx, val)
        assert ui.tolist() == ks
        if ks:
            np.testing.assert_array_equal(uv, np.stack(vs))
        # densify(coalesce(g)) == densify(g); idempotent; never grows
        np.testing.assert_array_equal(sparse.densify(ui, uv, 12), sparse.densify(idx, val, 12))
        ui2, uv2, _ = sparse.coalesce(ui, uv)
        assert ui2.tolist() == ui.tolist() and np.array_equal(uv2, uv)
        assert ui.size <= idx.size


def test_index_select_examples():
    g = GOLD["index_select"]
    ui = np.array(g["idx"])
    uv = np.arange(len(ui) * 2, dtype=np.float64).reshape(-1, 2)
    si, sv = sparse.index_select(ui, uv, set(g["keep"]))
    assert si.tolist() == g["out_idx"] and sv.tolist() == [[2.0, 3.0]]
    si, _ = sparse.index_select(ui, uv, set(g["idx"]))
    assert si.tolist() == g["idx"]
    si, _ = sparse.index_select(ui, uv, {7})
    assert si.size == 0


def test_densify_and_scatter_add_examples():
    for c in GOLD["densify"]["cases"]:
        assert sparse.densify(c["idx"], c["val"], c["rows"]).tolist() == c["out"]
    s = GOLD["scatter_add"]
    assert sparse.scatter_add(s["target"], s["idx"], s["val"], s["scale"]).tolist() == s["out"]
    with pytest.raises(IndexError):
        sparse.densify([5], [[1.0]], 3)


# ---------------------------------------------------------------- partition
def test_partition_examples_and_reassembly():
    for c in GOLD["partition"]["cases"]:
        assert [list(x) for x in partition.column_ranges(c["D"], c["N"])] == c["cols"]
    W = np.arange(4 * 5, dtype=np.float64).reshape(4, 5)
    for N in (1, 2, 3, 5):
        np.testing.assert_array_equal(np.hstack(partition.partition_columnwise(W, N)), W)
    with pytest.raises(ValueError):
        partition.column_ranges(3, 4)


def test_shard_lookup_tiling_and_balance():
    rng = np.random.default_rng(4)
    W = rng.standard_normal((50, 8))
    tokens = rng.integers(0, 50, 37)
    shards = partition.partition_columnwise(W, 4)
    np.testing.assert_array_equal(np.hstack([partition.shard_lookup(s, tokens) for s in shards]), W[tokens])
    assert partition.shard_lookup(shards[0], []).shape == (0, 2)
    with pytest.raises(IndexError):
        partition.shard_lookup(shards[0], [50])
    # column-wise: equal requests per shard; row-wise under Zipf: unequal
    from synthetic.workloads import zipf_ids
    z = zipf_ids(np.random.default_rng(5), 4000, 1000, 1.0)
    assert len(set(partition.request_counts_columnwise(z, 4))) == 1
    rc = partition.request_counts_rowwise(z, 1000, 4)
    assert sum(rc) == z.size and max(rc) > 2 * min(rc)


# ---------------------------------------------------------------- collectives
def test_collective_examples():
    a = GOLD["all_reduce"]
    out = collectives.all_reduce([np.array(x, np.float64) for x in a["inputs"]])
    assert all(o.tolist() == a["out"] for o in out)
    t = GOLD["all_to_all"]
    assert collectives.all_to_all(t["inputs"]) == t["out"]
    mb = GOLD["measure_bytes"]
    c = mb["alltoall_N4_block_m"]
    blocks = [[np.zeros(c["m"])] * c["N"] for _ in range(c["N"])]
    assert collectives.alltoall_sent_elems(blocks) == [c["sent_each"]] * c["N"]
    c = mb["allgather_N3_payload_m"]
    assert collectives.allgather_sent_elems([np.zeros(c["m"])] * c["N"]) == [c["sent_each"]] * c["N"]
    assert collectives.alltoall_sent_elems([[np.zeros(9)]]) == [0]  # N = 1


def test_alltoall_is_block_transpose_and_involution():
    rng = random.Random(6)
    for N in (2, 3, 4, 8):
        blocks = [[(r, s, rng.random()) for s in range(N)] for r in range(N)]
        out = collectives.all_to_all(blocks)
        for r in range(N):
            for s in range(N):
                assert out[s][r] == blocks[r][s]
        assert collectives.all_to_all(out) == blocks


def test_all_reduce_matches_single_process_sum():
    rng = np.random.default_rng(7)
    for N in (2, 3, 4, 8):
        xs = [rng.standard_normal(17) for _ in range(N)]
        out = collectives.all_reduce(xs)
        ref = xs[0].copy()
        for x in xs[1:]:
            ref = ref + x
        for o in out:
            np.testing.assert_array_equal(o, ref)


# ---------------------------------------------------------------- cost (Table 2)
def test_cost_worked_numbers():
    c = GOLD["cost"]
    assert cost.cost_allreduce(c["N"], c["M"], c["B"], c["beta"]) == pytest.approx(c["allreduce"])
    assert cost.cost_ps(c["N"], c["S"], c["alpha"], c["M"], c["B"], c["beta"]) == pytest.approx(c["ps"])
    assert cost.cost_allgather(c["N"], c["alpha"], c["M"], c["B"], c["beta"]) == pytest.approx(c["allgather"])
    assert cost.cost_alltoall(c["N"], c["alpha"], c["M"], c["B"], c["beta"]) == pytest.approx(c["alltoall"])
    assert cost.beta_threshold_allgather_vs_alltoall(c["N"], c["alpha"], c["M"], c["B"]) == pytest.approx(c["beta_threshold"])


def test_cost_sweep_alltoall_le_allreduce():
    rng = np.random.default_rng(8)
    for _ in range(10000):
        N = int(rng.integers(2, 257))
        a = float(rng.uniform(1e-6, 1.0))
        M, B, b = float(rng.uniform(1, 1e9)), float(rng.uniform(1, 1e9)), float(rng.uniform(0, 1))
        assert cost.cost_alltoall(N, a, M, B, b) <= cost.cost_allreduce(N, M, B, b) * (1 + 1e-12) + 1e-12
        assert cost.cost_alltoall(1, a, M, B, b) == 0.0
    # alpha = 1: AlltoAll and AllReduce coincide
    assert cost.cost_alltoall(8, 1.0, 1e6, 1e3, 0.1) == pytest.approx(cost.cost_allreduce(8, 1e6, 1e3, 0.1))
    # byte numerator of one AlltoAll equals the executed traffic (uniform case)
    N, m = 4, 12
    blocks = [[np.zeros(m // N)] * N for _ in range(N)]
    assert collectives.alltoall_sent_elems(blocks)[0] == cost.alltoall_bandwidth_numerator(N, m)


# ---------------------------------------------------------------- schedule
def test_vertical_split_worked_and_degenerate():
    g = GOLD["vertical_split"]
    idx = np.array(g["D_cur_n"])
    val = np.ones((idx.size, 2))
    (pi, pv), (di, dv), ip, isch = schedule.vertical_split(idx, val, [[9], idx], g["D_next"], 1)
    assert pi.tolist() == g["prior"] and di.tolist() == g["scheduled"]
    assert pv.tolist() == [[2.0, 2.0]]
    # full overlap -> scheduled empty; no overlap -> prior empty
    (_, _), (di, _), _, _ = schedule.vertical_split(idx, val, [idx], [1, 2, 5, 7], 0)
    assert di.size == 0
    (pi, _), (_, _), _, _ = schedule.vertical_split(idx, val, [idx], [], 0)
    assert pi.size == 0
    with pytest.raises(ValueError):
        schedule.vertical_split(idx, val, [idx], [], 3)


def test_vertical_split_brute_force_10k():
    rng = np.random.default_rng(9)
    for _ in range(10000):
        N = int(rng.integers(1, 5))
        D_cur = [rng.integers(0, 20, int(rng.integers(0, 12))) for _ in range(N)]
        n = int(rng.integers(0, N))
        D_next = rng.integers(0, 20, int(rng.integers(0, 12)))
        G_idx = D_cur[n]
        G_val = rng.integers(-3, 4, (G_idx.size, 2)).astype(np.float64)
        (pi, pv), (di, dv), ip, isch = schedule.vertical_split(G_idx, G_val, D_cur, D_next, n)
        # brute force by plain set logic + dict accumulation
        ks, vs = _dict_coalesce(G_idx, G_val)
        nxt = set(int(x) for x in D_next)
        assert pi.tolist() == [k for k in ks if k in nxt]
        assert di.tolist() == [k for k in ks if k not in nxt]
        assert set(pi.tolist()).isdisjoint(di.tolist())
        dense = sparse.densify(pi, pv, 20) + sparse.densify(di, dv, 20)
        np.testing.assert_array_equal(dense, sparse.densify(G_idx, G_val, 20))
        assert pi.size <= len(ks) <= G_idx.size


def test_issue_order_examples():
    q = GOLD["queue"]
    assert schedule.issue_order(q["priorities"], window=len(q["priorities"])) == q["drain_seq"]
    assert schedule.issue_order([5, 5, 5, 5], window=4) == [0, 1, 2, 3]        # FIFO ties
    assert schedule.issue_order([3, 1, 2, 0], window=1) == [0, 1, 2, 3]        # W=1: FIFO
    # W=2: after 2 arrivals issue min; [3,1] -> issue 1 (p=1); +2 -> {3,2}: issue 2; +0 -> {3,0}: 3; flush 0
    assert schedule.issue_order([3, 1, 2, 0], window=2) == [1, 2, 3, 0]


def test_issue_order_brute_force():
    rng = random.Random(10)
    for _ in range(2000):
        n = rng.randint(0, 12)
        pr = [rng.randint(-3, 3) for _ in range(n)]
        W = rng.randint(1, 14)
        out = schedule.issue_order(pr, W)
        assert sorted(out) == list(range(n))
        if W >= n:
            assert out == sorted(range(n), key=lambda s: (pr[s], s))
        if W == 1:
            assert out == list(range(n))


def test_prefetch_window():
    p = GOLD["prefetch"]
    assert [list(x) for x in schedule.prefetch_window(p["batches"])] == p["pairs"]
    assert list(schedule.prefetch_window(["b1"])) == [("b1", None)]


# ---------------------------------------------------------------- optimizers
def test_adam_step1_closed_form():
    # m = v = 0, t = 1:  dW = -lr * g / (|g| + eps / sqrt(1 - beta2))   (derived)
    rng = np.random.default_rng(11)
    g = rng.standard_normal((5, 7)) * 10.0 ** rng.integers(-9, 2, (5, 7))
    W = rng.standard_normal((5, 7))
    m, v = np.zeros_like(W), np.zeros_like(W)
    W0 = W.copy()
    lr, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    optim.adam_apply(W, m, v, np.arange(5), g, 1, lr, b1, b2, eps)
    np.testing.assert_allclose(W - W0, -lr * g / (np.abs(g) + eps / np.sqrt(1 - b2)), rtol=1e-12, atol=1e-15)  # W - W0 cancels: |W| ~ 1
    np.testing.assert_allclose(m, (1 - b1) * g, rtol=1e-15)
    np.testing.assert_allclose(v, (1 - b2) * g * g, rtol=1e-15)


def test_adam_matches_torch_sparse_adam():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(12)
    L, D = 20, 6
    W0 = rng.standard_normal((L, D))
    p = torch.nn.Parameter(torch.tensor(W0, dtype=torch.float64))
    opt = torch.optim.SparseAdam([p], lr=1e-2, betas=(0.8, 0.99), eps=1e-6)
    W, m, v = W0.copy(), np.zeros((L, D)), np.zeros((L, D))
    for t in range(1, 5):
        rows = np.unique(rng.integers(0, L, 8))
        g = rng.standard_normal((rows.size, D))
        p.grad = torch.sparse_coo_tensor(torch.tensor(rows[None, :]), torch.tensor(g), (L, D))
        opt.step()
        optim.adam_apply(W, m, v, rows, g, t, 1e-2, 0.8, 0.99, 1e-6)
        np.testing.assert_allclose(W, p.detach().numpy(), rtol=1e-13, atol=1e-15)


def test_partial_adam_two_parts_bitwise_equal_to_one():
    rng = np.random.default_rng(13)
    for _ in range(1000):
        L, D = 30, 4
        W0 = rng.standard_normal((L, D))
        rows = np.unique(rng.integers(0, L, 12))
        g = rng.standard_normal((rows.size, D))
        cut = rng.random(rows.size) < 0.5
        a = optim.PartialAdam(lr=1e-3)
        Wa, ma, va = W0.copy(), np.zeros((L, D)), np.zeros((L, D))
        a.apply_partial(Wa, ma, va, rows, g, True)
        b = optim.PartialAdam(lr=1e-3)
        Wb, mb, vb = W0.copy(), np.zeros((L, D)), np.zeros((L, D))
        b.apply_partial(Wb, mb, vb, rows[cut], g[cut], False)
        b.apply_partial(Wb, mb, vb, rows[~cut], g[~cut], True)
        assert np.array_equal(Wa, Wb) and np.array_equal(ma, mb) and np.array_equal(va, vb)
        assert a.step == b.step == 1
    # overlapping parts are rejected
    c = optim.PartialAdam()
    Wc, mc, vc = np.zeros((3, 1)), np.zeros((3, 1)), np.zeros((3, 1))
    c.apply_partial(Wc, mc, vc, [0], np.ones((1, 1)), False)
    with pytest.raises(ValueError):
        c.apply_partial(Wc, mc, vc, [0], np.ones((1, 1)), True)


def test_partial_adam_empty_prior_only_scheduled_changes_state():
    W, m, v = np.ones((4, 2)), np.zeros((4, 2)), np.zeros((4, 2))
    a = optim.PartialAdam()
    a.apply_partial(W, m, v, np.zeros(0, np.int64), np.zeros((0, 2)), False)
    assert np.array_equal(W, np.ones((4, 2))) and a.step == 0
    a.apply_partial(W, m, v, [1], np.ones((1, 2)), True)
    assert a.step == 1 and W[1, 0] != 1.0 and W[0, 0] == 1.0


def test_sgd_matches_dense_step():
    rng = np.random.default_rng(14)
    W = rng.standard_normal((10, 3))
    rows = np.array([1, 4, 7])
    g = rng.standard_normal((3, 3))
    dense = np.zeros((10, 3))
    dense[rows] = g
    ref = W - 0.1 * dense            # a dense-gradient SGD step
    optim.sgd_apply(W, rows, g, 0.1)
    np.testing.assert_array_equal(W, ref)


# ---------------------------------------------------------------- NEXT-4: sparse Adagrad

def test_adagrad_matches_torch_adagrad_sparse():
    """oracle.optim.adagrad_apply against torch.optim.Adagrad on sparse
    gradients (a library routine, independent of the oracle's code)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(21)
    L, D = 20, 6
    W0 = rng.standard_normal((L, D))
    p = torch.nn.Parameter(torch.tensor(W0, dtype=torch.float64))
    opt = torch.optim.Adagrad([p], lr=5e-2, eps=1e-10)
    W, s = W0.copy(), np.zeros((L, D))
    for _ in range(5):
        rows = np.unique(rng.integers(0, L, 8))
        g = rng.standard_normal((rows.size, D))
        p.grad = torch.sparse_coo_tensor(torch.tensor(rows[None, :]), torch.tensor(g), (L, D))
        opt.step()
        optim.adagrad_apply(W, s, rows, g, 5e-2, 1e-10)
        np.testing.assert_allclose(W, p.detach().numpy(), rtol=1e-13, atol=1e-15)


def test_adagrad_step1_closed_form_and_parts():
    """Step 1 from s = 0: dW = -lr g / (|g| + eps) (a sign step); two disjoint
    parts equal one call bitwise (element-wise optimizer)."""
    rng = np.random.default_rng(22)
    L, D = 12, 4
    W = rng.uniform(-1, 1, (L, D))
    g = rng.uniform(-1, 1, (L, D))
    rows = np.arange(L)
    W1, s1 = W.copy(), np.zeros((L, D))
    optim.adagrad_apply(W1, s1, rows, g, 0.1, 1e-10)
    np.testing.assert_allclose(W1 - W, -0.1 * g / (np.abs(g) + 1e-10), rtol=1e-14)
    W2, s2 = W.copy(), np.zeros((L, D))
    optim.adagrad_apply(W2, s2, rows[:5], g[:5], 0.1, 1e-10)
    optim.adagrad_apply(W2, s2, rows[5:], g[5:], 0.1, 1e-10)
    assert np.array_equal(W1, W2) and np.array_equal(s1, s2)


@pytest.mark.parametrize("mode", ["raw", "coal", "split"])
def test_adagrad_exchange_equals_dense_reference(mode):
    """The simulated N-worker exchange with Adagrad reaches the plain definition
    (dense scatter-add, one Adagrad step on the touched rows)."""
    from oracle import exchange, partition
    from synthetic import get_config, make_workload
    from synthetic.workloads import gen_table
    cfg = get_config("tiny")
    wl = make_workload(cfg, 2, 3)
    W = gen_table(cfg).astype(np.float64)
    opt = exchange.OptimConfig("adagrad", lr=0.05, eps=1e-10)
    shards = partition.partition_columnwise(W.copy(), 2)
    s_sh = [np.zeros_like(x) for x in shards]
    Wd, sd = W.copy(), np.zeros_like(W)
    for k in range(2):
        exchange.simulate_iteration(shards, wl.ids[k], wl.dY[k], wl.ids[k + 1], k + 1, mode, "fp64", opt, s_sh, None)
        exchange.dense_reference(Wd, wl.ids[k], wl.dY[k], k + 1, "fp64", opt, sd, None)
    np.testing.assert_allclose(np.hstack(shards), Wd, rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.hstack(s_sh), sd, rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- NEXT-4: row-wise partition (load-imbalance study)

def test_rowwise_vs_columnwise_requests_worked_example():
    """row-wise shards get unequal request counts when word
    frequencies differ; column-wise shards all serve every request."""
    from oracle import partition
    toks = np.array([0, 0, 0, 1, 5])
    assert partition.request_counts_rowwise(toks, 6, 2) == [4, 1]          # rows [0,3) and [3,6)
    assert partition.request_counts_rowwise_hashed(toks, 2) == [3, 2]      # even / odd ids
    assert partition.request_counts_columnwise(toks, 2) == [5, 5]
    ids_all = [np.array([0, 0, 1]), np.array([0, 5])]
    # column: owner 0 sends rank 1's 2 tokens, owner 1 sends rank 0's 3 tokens, D/N = 2 columns of 4 B
    assert partition.forward_bytes_out(ids_all, 6, 4, 2, "column") == [2 * 2 * 4, 3 * 2 * 4]
    # row: owner 0 (rows 0..2) sends rank 1's id 0; owner 1 (rows 3..5) sends nothing of rank 0's
    assert partition.forward_bytes_out(ids_all, 6, 4, 2, "row") == [1 * 4 * 4, 0]


def test_rowwise_imbalance_on_zipf_batches():
    """On Zipf-distributed (frequency-sorted) ids the most loaded row-wise owner
    serves far more than the mean, column-wise owners exactly the mean."""
    from oracle import partition
    from synthetic import get_config, make_workload
    cfg = get_config("gnmt")
    N = 4
    wl = make_workload(cfg, N, 1, with_dY=False)
    ids = wl.ids[0]
    col = partition.forward_bytes_out(ids, cfg.L, cfg.D, N, "column", 2)
    row = partition.forward_bytes_out(ids, cfg.L, cfg.D, N, "row", 2)
    assert max(col) / (sum(col) / N) < 1.01
    assert max(row) / (sum(row) / N) > 2.0
