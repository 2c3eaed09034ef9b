"""In-box baselines (baselines/inbox.py): the
Horovod-AllGather-style and dense-AllReduce aggregations reach the same update
as the oracle's plain hybrid exchange (RAW mode: no wire rounding), free-running
with the accumulated sigma metric (tests/_metric.py).  Single rank here (the
collectives are identities); the multi-rank runs are bench measurements."""

import dataclasses

import numpy as np
import pytest

from oracle import exchange, partition
from synthetic import get_config, make_workload
from synthetic.workloads import gen_table

from _metric import SigmaAcc, assert_close_acc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["allgather", "allreduce"])
@pytest.mark.parametrize("name", ["tiny", "gnmt"])
def test_inbox_baseline_matches_oracle(kind, name):
    import torch
    from baselines.inbox import ReplicatedTable
    cfg = get_config(name) if name == "tiny" else dataclasses.replace(get_config(name), batch=8)
    wl = make_workload(cfg, 1, 4)
    W = gen_table(cfg)
    dev = torch.device("cuda", 0)
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    rt = ReplicatedTable(torch.from_numpy(W).to(dev).to(tdt), optim=cfg.optim, lr=cfg.lr, world=1, kind=kind)
    shards = partition.partition_columnwise(W.astype(np.float64), 1)
    m = [np.zeros_like(shards[0])] if cfg.optim == "adam" else None
    v = [np.zeros_like(shards[0])] if cfg.optim == "adam" else None
    opt = exchange.OptimConfig(cfg.optim, lr=cfg.lr)
    acc = SigmaAcc(cfg.D)
    for k in range(3):
        ids = torch.from_numpy(wl.ids[k][0].astype(np.int64)).to(dev)
        Y = rt.forward(ids)
        dY = torch.from_numpy(wl.dY[k][0]).to(dev).to(tdt)
        rt.backward(ids, dY, cfg.max_tokens)
        res = exchange.simulate_iteration(shards, wl.ids[k], wl.dY[k], wl.ids[k + 1], k + 1, "raw", cfg.dtype, opt,
                                          m, v)
        snap = acc.snapshot()
        acc.add(res.U, res.sigma_W)
        gY = Y.double().cpu().numpy()
        assert_close_acc(gY, res.Y[0], snap.get(wl.ids[k][0]), cfg.dtype, f"{kind} iter {k + 1} Y")
        rows = acc.ids
        gW = rt.W[torch.from_numpy(rows).to(dev)].double().cpu().numpy()
        assert_close_acc(gW, shards[0][rows], acc.get(rows), cfg.dtype, f"{kind} iter {k + 1} W")
