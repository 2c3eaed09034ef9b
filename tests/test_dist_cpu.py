"""World-size-2 gloo tests (CPU) of the multi-process host logic: the
bootstrap exchange of IPC handles / NCCL id, per-rank workload generation and
column-shard assignment are consistent across ranks, and the oracle's
simulated exchange agrees with each rank's local view."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2110_09132_b200.runtime import broadcast_bytes, exchange_bytes
        from oracle import exchange, partition
        from synthetic import get_config, make_workload
        from synthetic.workloads import gen_ids, gen_table

        # 1. handle all-gather keeps rank order; unique-id broadcast reaches everyone
        fake = bytes([rank]) * 64
        got = exchange_bytes(fake, world)
        assert [g[0] for g in got] == list(range(world)) and all(len(g) == 64 for g in got)
        nid = broadcast_bytes(b"\x07" * 128 if rank == 0 else None, world)
        assert nid == b"\x07" * 128

        # 2. every rank regenerates the same global workload (inputs are a pure function of the seed)
        cfg = get_config("tiny")
        mine = gen_ids(cfg, 0, rank)
        allv = [None] * world
        dist.all_gather_object(allv, mine.tolist())
        wl = make_workload(cfg, world, 2)
        for r in range(world):
            assert allv[r] == wl.ids[0][r].tolist()

        # 3. column shard of this rank == the oracle partition's shard r; hconcat of the
        #    gathered shards reproduces W
        W = gen_table(cfg)
        d = cfg.D // world
        shard = W[:, rank * d:(rank + 1) * d]
        shards = [None] * world
        dist.all_gather_object(shards, shard)
        assert np.array_equal(np.hstack(shards), W)
        assert np.array_equal(partition.partition_columnwise(W, world)[rank], shard)

        # 4. each rank's forward rows (oracle, simulated) == its local dense lookup
        res = exchange.simulate_iteration(partition.partition_columnwise(W.astype(np.float64), world),
                                          wl.ids[0], wl.dY[0], wl.ids[1], 1, "split", "fp64",
                                          exchange.OptimConfig("sgd", lr=0.1))
        assert np.array_equal(res.Y[rank], W.astype(np.float64)[wl.ids[0][rank]])
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert res == [(0, "ok"), (1, "ok")], res
