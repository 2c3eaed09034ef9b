"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same
seeded inputs.  Integers bit-exact, forward rows exact, updated state within
the sigma-normalised tolerance (1e-5 fp32 / 2e-2 bf16)."""

import dataclasses

import numpy as np
import pytest

from synthetic import get_config
from synthetic.workloads import Config

from _harness import graph_parity, parity_run

pytestmark = pytest.mark.gpu


def _small(name, **kw):
    """A config with the paper-shaped vocabulary/width of `name` and a
    reduced batch, so the oracle finishes in seconds while the batch still
    spans many chunks, segments and a ragged tail."""
    return dataclasses.replace(get_config(name), **kw)


@pytest.mark.parametrize("mode", ["raw", "coal", "split"])
def test_tiny_sgd_modes(mode):
    parity_run(get_config("tiny"), N=1, mode=mode, iters=4)


def test_tiny_pad_dropped():
    parity_run(get_config("tiny"), N=1, mode="split", iters=3, pad_id=0)


def test_tiny_adam_split():
    parity_run(get_config("tiny"), N=1, mode="split", iters=4, optim="adam", lr=1e-2)


def test_tiny_no_prefetch_last_step_each_time():
    # next_ids only on the first step; last step has D_next = ∅ (everything scheduled)
    parity_run(get_config("tiny"), N=1, mode="split", iters=2, last_none=True)


@pytest.mark.parametrize("name", ["gnmt", "transformer", "bert_large"])
@pytest.mark.parametrize("mode", ["raw", "split"])
def test_bf16_configs_small_batch(name, mode):
    cfg = get_config(name)
    small = _small(name, batch=8) if not cfg.packed else _small(name, seq_len=600)
    parity_run(small, N=1, mode=mode, iters=3)


def test_lm_fp32_adam_small_batch():
    parity_run(_small("lstm_lm", batch=16), N=1, mode="split", iters=3)


@pytest.mark.slow
def test_lm_full_size_split_adam():
    """BASELINE configs[1] at full size, the configuration bench.py times."""
    parity_run(get_config("lstm_lm"), N=1, mode="split", iters=2, rows_sample=20000)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["gnmt", "transformer", "bert_large"])
def test_bf16_full_size_split(name):
    parity_run(get_config(name), N=1, mode="split", iters=2)


def test_long_zipf_head_segments():
    """Heavy duplication: a segment of ~1000 rows (pad) and the Zipf head span
    many reduce chunks (two-level combine path)."""
    cfg = Config("dup", 64, 256, "fp32", 64, 40, 2, optim="sgd", lr=0.1, zipf_s=1.6)
    parity_run(cfg, N=1, mode="coal", iters=3)
    parity_run(cfg, N=1, mode="raw", iters=2)


def test_single_token_and_full_capacity_batches():
    cfg = Config("one", 50, 32, "fp32", 1, 1, 1, optim="sgd", lr=0.5)
    parity_run(cfg, N=1, mode="split", iters=3)
    cfg = Config("cap", 3000, 64, "bf16", 64, 256, 256, optim="adam", lr=1e-3)  # every slot used (no pad)
    parity_run(cfg, N=1, mode="split", iters=2)


def test_errors_id_range_and_state():
    import torch
    from paper_2110_09132_b200 import embrace as E
    from paper_2110_09132_b200.runtime import EmbraceExchange
    dev = torch.device("cuda", 0)
    W = torch.zeros(100, 16, device=dev)
    ex = EmbraceExchange(100, 16, W, max_tokens=32, mode="split")
    ids = torch.tensor([1, 2, 100], dtype=torch.int32, device=dev)     # 100 is out of range
    ex.forward(ids)
    ex.backward(torch.zeros(3, 16, device=dev), None)
    with pytest.raises(E.EmbError) as ei:
        ex.flush()
    assert ei.value.name == "EMB_ERR_ID_RANGE"
    ex.close()
    ex = EmbraceExchange(100, 16, W, max_tokens=32, mode="split")
    a = torch.tensor([1, 2, 3], dtype=torch.int32, device=dev)
    ex.forward(a)
    ex.backward(torch.zeros(3, 16, device=dev), a + 1)                    # promise [2, 3, 4] ...
    ex.forward(a)                                                        # ... but send [1, 2, 3]
    ex.backward(torch.zeros(3, 16, device=dev), None)
    with pytest.raises(E.EmbError) as ei:
        ex.flush()
    assert ei.value.name == "EMB_ERR_STATE"
    ex.close()
    # host-side checks fail before anything is enqueued
    ex = EmbraceExchange(100, 16, W, max_tokens=4, mode="coal")
    with pytest.raises(E.EmbError) as ei:
        ex.forward(torch.zeros(5, dtype=torch.int32, device=dev))
    assert ei.value.name == "EMB_ERR_CAPACITY"
    with pytest.raises(E.EmbError) as ei:
        ex.backward(torch.zeros(1, 16, device=dev))
    assert ei.value.name == "EMB_ERR_STATE"
    ex.close()


def test_empty_batch():
    import torch
    from paper_2110_09132_b200.runtime import EmbraceExchange
    dev = torch.device("cuda", 0)
    W = torch.randn(64, 16, device=dev)
    ex = EmbraceExchange(64, 16, W.clone(), max_tokens=8, mode="split")
    e = torch.zeros(0, dtype=torch.int32, device=dev)
    out = ex.forward(e)
    ex.backward(torch.zeros(0, 16, device=dev), e)
    ex.forward(e)
    ex.backward(torch.zeros(0, 16, device=dev), None)
    ex.flush()
    assert out.shape == (0, 16)
    assert torch.equal(ex.shard(), W)
    ex.close()


def test_run_twice_bitwise_deterministic():
    import torch
    from paper_2110_09132_b200.runtime import EmbraceExchange
    from synthetic import make_workload
    from synthetic.workloads import gen_table
    cfg = Config("det", 500, 128, "fp32", 32, 40, 4, optim="adam", lr=1e-3, zipf_s=1.3)
    wl = make_workload(cfg, 1, 4)
    W = torch.from_numpy(gen_table(cfg)).cuda()
    outs = []
    for _ in range(2):
        ex = EmbraceExchange(cfg.L, cfg.D, W.clone(), max_tokens=cfg.max_tokens, mode="split", optim="adam", lr=1e-3)
        for k in range(3):
            ex.forward(torch.from_numpy(wl.ids[k][0]).cuda())
            ex.backward(torch.from_numpy(wl.dY[k][0]).cuda(), torch.from_numpy(wl.ids[k + 1][0]).cuda())
        ex.flush()
        outs.append((ex.shard().clone(), ex.adam_m().clone(), ex.adam_v().clone()))
        ex.close()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_prefetch_split_adam():
    """emb_prefetch (the paper's prefetch as an early fork point) before every forward."""
    cfg = get_config("tiny")
    parity_run(cfg, N=1, mode="split", iters=4, optim="adam", lr=1e-3, prefetch=True)
    parity_run(dataclasses.replace(get_config("lstm_lm"), batch=16), N=1, mode="split", iters=3,
               rows_sample=512, prefetch=True)


# ---------------------------------------------------------------- round 2: free-running, pipelined, graph

def test_free_running_50_iterations_fp32_adam():
    """50 iterations with no resync: the oracle runs free, the tolerance is the
    sigma accumulated over the iterations that touched a row (tests/_metric.py),
    so the Adam step counter to t = 50 and every row's history are checked."""
    cfg = Config("free", 2000, 64, "fp32", 8, 24, 6, optim="adam", lr=1e-3, zipf_s=1.1)
    parity_run(cfg, N=1, mode="split", iters=50, free=True)


def test_free_running_bf16_adam():
    parity_run(_small("bert_large", batch=2), N=1, mode="split", iters=12, free=True)


@pytest.mark.parametrize("prefetch", [False, True])
def test_pipelined_n1_lm(prefetch):
    """LM-shaped, 6 iterations back to back without flush, NULL next_ids mid-run."""
    parity_run(_small("lstm_lm", batch=16), N=1, mode="split", iters=6, prefetch=prefetch, pipelined=True,
               null_at=(2,), rows_sample=1024)


@pytest.mark.parametrize("name", ["tiny", "gnmt"])
def test_graph_replay_n1(name):
    """The bench's timed path (CUDA graph of a cycle of steps, replayed) against the oracle."""
    cfg = get_config(name) if name == "tiny" else _small(name, batch=8)
    errs, iters = graph_parity(cfg, N=1)
    assert iters == 3 + 2 * 4 + 1


@pytest.mark.parametrize("rem", [1, 3])
def test_graph_split_cycle_n1(rem):
    """bench.py's short-run path: the cycle also captured as a graph of its first
    `rem` steps plus one of the rest (warmed as one cycle, closed after the
    timed replays), emb_prefetch inside the graphs — final state vs the oracle."""
    errs, iters = graph_parity(get_config("tiny"), N=1, nb=4, rem=rem, graph_prefetch=True)
    assert iters == 3 + (1 + 1 + 2 + 1) * 4 + 1  # warm cycle, warm split cycle, 2 replays, closing split cycle


@pytest.mark.slow
def test_graph_replay_lm_full_size():
    """BASELINE configs[1] at full size through the graph path bench.py times."""
    graph_parity(get_config("lstm_lm"), N=1, warm=3, nb=4, replays=2)


def test_backward_null_then_forward_no_flush():
    """backward(next_ids = NULL) followed by forward without a
    flush in between must not lose the next batch's gradient."""
    parity_run(get_config("tiny"), N=1, mode="split", iters=5, null_at=(0, 1, 2), pipelined=True)


# ---------------------------------------------------------------- NEXT-4: sparse Adagrad

@pytest.mark.parametrize("mode", ["raw", "coal", "split"])
def test_adagrad_tiny(mode):
    parity_run(get_config("tiny"), N=1, mode=mode, iters=4, optim="adagrad", lr=0.05)


def test_adagrad_bf16_paper_shape_free_running():
    parity_run(_small("gnmt", batch=8), N=1, mode="split", iters=6, optim="adagrad", lr=1e-2, free=True)


# ---------------------------------------------------------------- NEXT-3: several tables, one exchange

def _two_tables(L1):
    """ids override: each rank's first half looks up table A (rows [0, L1)), the
    second half table B (rows [L1, L)): global row ids, as embrace.h prescribes."""
    def f(ids):
        out = []
        for it in ids:
            row = []
            for x in it:
                x = np.asarray(x, np.int64).copy()
                h = x.size // 2
                x[:h] = x[:h] % L1
                x[h:] = L1 + (x[h:] % (1000 - L1))
                row.append(x.astype(np.int32))
            out.append(row)
        return out
    return f


@pytest.mark.parametrize("prefetch", [False, True])
def test_two_tables_one_exchange(prefetch):
    cfg = Config("twotab", 1000, 16, "fp32", 8, 16, 8, optim="adam", lr=1e-2)
    parity_run(cfg, N=1, mode="split", iters=4, ids_override=_two_tables(600), table_rows=(600, 400),
               prefetch=prefetch)


def test_forward_dedup_n1_knob(monkeypatch):
    """EMB_FWD_DEDUP1=1: the N == 1 forward gathers each distinct row once per
    reduce chunk (measured slower, default off): Y still exact."""
    monkeypatch.setenv("EMB_FWD_DEDUP1", "1")
    parity_run(get_config("tiny"), N=1, mode="split", iters=4, prefetch=True)
    parity_run(_small("lstm_lm", batch=8), N=1, mode="split", iters=3, prefetch=True, rows_sample=512)


@pytest.mark.parametrize("bulk", ["0", "1"])
def test_forward_bulk_copy_knob(monkeypatch, bulk):
    """EMB_FWD_BULK forces the N == 1 forward onto the bulk-copy (TMA) gather or
    the register gather (default: bulk for tables > 96 MB).  Both exact, fp32
    and bf16, ragged batch tails, with and without the prefetched sort."""
    monkeypatch.setenv("EMB_FWD_BULK", bulk)
    parity_run(get_config("tiny"), N=1, mode="split", iters=3, prefetch=False)
    parity_run(_small("gnmt", batch=5), N=1, mode="split", iters=3, prefetch=True)
    parity_run(_small("lstm_lm", batch=3), N=1, mode="coal", iters=2, prefetch=True, rows_sample=512)


# ---------------------------------------------------------------- tokens per rank above 16384 (16-CTA sort)

def test_batch_above_16k_tokens():
    """max_tokens up to 32768 (the 16-CTA cluster sort): GNMT shape with 8x its
    batch (26,624 tokens per rank) and an LM-vocabulary fp32 case."""
    parity_run(dataclasses.replace(get_config("gnmt"), batch=1024), N=1, mode="split", iters=2, prefetch=True)
    parity_run(dataclasses.replace(get_config("lstm_lm"), batch=512), N=1, mode="coal", iters=2, rows_sample=1024)
