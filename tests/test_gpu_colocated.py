"""Every N > 1 code path on ONE GPU: N co-located ranks (one process, N
emb_ctx on the same device, embrace.h emb_shard_init_colocated) run the same
kernels, flag gates and peer loads / stores as N GPUs over NVLink — the id
all-gather push, the forward pull (and its dedup), the gradient push to the
owners' receive rows, the owner merge, the scheduled part on the side stream.
Each rank's outputs are compared with the oracle's simulated N workers
(tests/_harness.py): Y and every integer intermediate exactly, the shards /
m / v with the sigma metric."""

import dataclasses
import os

import pytest

from synthetic import get_config

from _harness import graph_parity, parity_run

pytestmark = pytest.mark.gpu


def _small(name, batch):
    cfg = get_config(name)
    if cfg.packed:
        return dataclasses.replace(cfg, seq_len=batch * 40)
    return dataclasses.replace(cfg, batch=batch)


def test_connections_env():
    assert int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8")) >= 32


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("mode", ["raw", "coal", "split"])
def test_tiny_colocated(n, mode):
    parity_run(get_config("tiny"), N=n, mode=mode, iters=3, colocated=True)


@pytest.mark.parametrize("n", [2, 4])
def test_tiny_adam_prefetch_colocated(n):
    parity_run(get_config("tiny"), N=n, mode="split", iters=4, optim="adam", lr=1e-2, prefetch=True,
               colocated=True)


def test_pad_dropped_colocated():
    parity_run(_small("gnmt", 16), N=2, mode="split", iters=3, pad_id=0, colocated=True)


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("name", ["gnmt", "transformer", "bert_large"])
def test_bf16_paper_shapes_colocated(n, name):
    parity_run(_small(name, 4 if name == "bert_large" else 16), N=n, mode="split", iters=3, colocated=True)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_lm_colocated(n):
    parity_run(_small("lstm_lm", 16), N=n, mode="split", iters=2, rows_sample=2048, colocated=True)


@pytest.mark.parametrize("mode", ["raw", "coal"])
def test_modes_n8_colocated(mode):
    parity_run(_small("gnmt", 8), N=8, mode=mode, iters=2, colocated=True)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_prefetch_paper_shape_colocated(n):
    parity_run(_small("bert_large", 2), N=n, mode="split", iters=3, prefetch=True, colocated=True)


@pytest.mark.parametrize("n", [1, 2, 4])
@pytest.mark.parametrize("prefetch", [False, True])
def test_pipelined_null_mid_run(n, prefetch):
    """K iterations back to back with no flush between them (the overlap of the
    scheduled part of t with forward(t+1), parity double buffers, side-stream
    work), a NULL next_ids in the middle followed by a forward (a
    late prefetch copy must not clobber the next forward's count), then every
    Y and the final state against the free-running oracle."""
    cfg = get_config("tiny") if n < 8 else _small("gnmt", 4)
    parity_run(cfg, N=n, mode="split", iters=8, optim="adam", lr=1e-2, prefetch=prefetch, colocated=n > 1,
               pipelined=True, null_at=(2, 5))


@pytest.mark.parametrize("n", [2, 8])
def test_pipelined_paper_shape(n):
    parity_run(_small("gnmt", 8), N=n, mode="split", iters=6, prefetch=True, colocated=True, pipelined=True,
               null_at=(3,))


def test_graph_replay_colocated():
    """The bench's CUDA-graph cycle, two co-located ranks, replayed twice."""
    graph_parity(_small("gnmt", 8), N=2, colocated=True)


def test_graph_split_cycle_colocated():
    """bench.py's short-run graph path (cycle split in rem + rest), two co-located ranks."""
    graph_parity(_small("gnmt", 8), N=2, colocated=True, rem=1, graph_prefetch=True)


@pytest.mark.parametrize("n", [2, 4])
def test_adagrad_colocated(n):
    parity_run(get_config("tiny"), N=n, mode="split", iters=3, optim="adagrad", lr=0.05, colocated=True)
    parity_run(_small("bert_large", 2), N=n, mode="split", iters=3, optim="adagrad", lr=1e-2, colocated=True)


def test_two_tables_colocated():
    """GNMT-like: encoder and decoder tables of one width in one exchange (NEXT-3)."""
    from synthetic.workloads import Config
    from test_gpu_parity import _two_tables
    cfg = Config("twotab", 1000, 64, "bf16", 8, 16, 8, optim="adam", lr=1e-2)
    parity_run(cfg, N=2, mode="split", iters=3, ids_override=_two_tables(600), table_rows=(600, 400),
               prefetch=True, colocated=True)


def test_batch_above_16k_colocated():
    parity_run(_small("transformer", 600), N=2, mode="split", iters=2, prefetch=True, colocated=True)
