"""GPU-vs-oracle parity driver shared by the single-GPU tests, the multi-GPU
torchrun worker (tests/dist_worker.py) and __graft_entry__.smoke().

Each rank generates every rank's seeded inputs (synthetic/), runs its own part
of the exchange through the C ABI, runs the oracle for all N simulated
workers on the same arrays, and compares its own outputs:
  * Y (forward output)                      exact
  * gathered ids, slot lists, counts, perm  exact (integers)
  * shard rows, Adam m / v                  sigma-normalised (tests/_metric.py)
  * byte counters                           exact vs the S8 closed forms
"""

import numpy as np

from oracle import exchange, partition
from synthetic import make_workload
from synthetic.workloads import PAD_ID, gen_table

from _metric import assert_close


def _to_torch(x, dtype, device):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype == "bf16":
        t = t.to(torch.bfloat16)          # values are already on the bf16 grid: exact
    return t.to(device)


def _np64(t):
    import torch
    return t.detach().to(torch.float64).cpu().numpy()


def parity_run(cfg, N=1, rank=0, mode="split", iters=3, optim=None, lr=None, pad_id=-1, last_none=True,
               device=0, rows_sample=None, ids_override=None, check=True, report=None, prefetch=False):
    """Run `iters` iterations on this rank and assert parity after each.
    Returns a dict of max errors seen (for reporting)."""
    import torch
    from paper_2110_09132_b200 import embrace as E
    from paper_2110_09132_b200.runtime import EmbraceExchange

    dev = torch.device("cuda", device)
    torch.cuda.set_device(dev)
    optim = optim or cfg.optim
    lr = lr if lr is not None else cfg.lr
    wl = make_workload(cfg, N, iters + 1)
    if ids_override is not None:
        wl.ids = ids_override(wl.ids)
        wl.dY = [[np.asarray(wl.dY[k][r][: len(wl.ids[k][r])]) if len(wl.dY[k][r]) >= len(wl.ids[k][r])
                  else np.resize(wl.dY[k][r], (len(wl.ids[k][r]), cfg.D)).astype(np.float32)
                  for r in range(N)] for k in range(iters + 1)]
    W = gen_table(cfg)
    shards = partition.partition_columnwise(W, N)                     # oracle state (float32 grid values)
    m = [np.zeros_like(s) for s in shards] if optim == "adam" else None
    v = [np.zeros_like(s) for s in shards] if optim == "adam" else None
    opt = exchange.OptimConfig(optim, lr=lr)
    d = cfg.D // N
    max_tokens = max(cfg.max_tokens, max(len(x) for it in wl.ids for x in it))
    ex = EmbraceExchange(cfg.L, cfg.D, _to_torch(shards[rank], cfg.dtype, dev), world=N, rank=rank, device=device,
                         dtype=cfg.dtype, max_tokens=max_tokens, mode=mode, optim=optim, lr=lr, pad_id=pad_id)
    errs = {"W": 0.0, "m": 0.0, "v": 0.0}
    esz = 2 if cfg.dtype == "bf16" else 4
    fwd_bytes = np.zeros(N, np.int64)
    bwd_bytes = np.zeros(N, np.int64)
    try:
        for k in range(iters):
            t = k + 1
            nxt = None if (last_none and k == iters - 1) else wl.ids[k + 1]
            ids_t = _to_torch(wl.ids[k][rank].astype(np.int32), None, dev)
            dY_t = _to_torch(wl.dY[k][rank], cfg.dtype, dev)
            nxt_t = None if nxt is None else _to_torch(nxt[rank].astype(np.int32), None, dev)
            if prefetch and nxt_t is not None:
                ex.prefetch(nxt_t)  # emb_prefetch: the next batch's work forks before this forward
            Y = ex.forward(ids_t)
            ex.backward(dY_t, nxt_t)
            ex.flush()
            res = exchange.simulate_iteration(shards, wl.ids[k], wl.dY[k], nxt, t, mode, cfg.dtype, opt, m, v,
                                              pad_id)
            if not check:
                continue
            # ---- forward: exact
            gY = _np64(Y)
            if not np.array_equal(gY, res.Y[rank]):
                bad = np.argwhere(gY != res.Y[rank])[:5]
                raise AssertionError(f"iter {t}: forward Y differs at {bad.tolist()}")
            # ---- integers: exact
            cnts = ex.debug(E.EMB_DBG_COUNTS).reshape(N, 4)
            for n in range(N):
                ids_n = np.asarray(wl.ids[k][n], np.int64)
                assert np.array_equal(ex.debug(E.EMB_DBG_GIDS, n), ids_n), f"iter {t}: gathered ids of {n}"
                # perm: positions sorted by (dropped, id, position); dropped = pad when pad_id >= 0
                drop = (ids_n == pad_id) if pad_id >= 0 else np.zeros(ids_n.size, bool)
                want_perm = np.lexsort((np.arange(ids_n.size), ids_n, drop))
                got_perm = ex.debug(E.EMB_DBG_PERM, n)
                if not np.array_equal(got_perm, want_perm):
                    bad = np.flatnonzero(got_perm != want_perm)[:6] if got_perm.size == want_perm.size else []
                    raise AssertionError(f"iter {t}: perm of {n}: sizes {got_perm.size}/{want_perm.size}, "
                                         f"first diffs at {list(bad)}: got {got_perm[bad]} want {want_perm[bad]}; "
                                         f"ids there {ids_n[want_perm[bad]]} / {ids_n[got_perm[bad]]}")
                want = np.concatenate([res.P_n[n], res.D_n[n]]).astype(np.int64)
                got = ex.debug(E.EMB_DBG_SLOT_IDS, n)
                assert np.array_equal(got, want), f"iter {t}: slot ids of source {n}: {got[:8]} vs {want[:8]}"
                assert cnts[n, 0] == len(ids_n) and cnts[n, 1] == res.u[n] and cnts[n, 2] == res.p[n], \
                    f"iter {t}: counts of {n}: {cnts[n]} vs T={len(ids_n)} u={res.u[n]} p={res.p[n]}"
            st = ex.stats()
            assert st["err_flags"] == 0, f"device error flags {st['err_flags']}"
            # ---- byte counters (S8): pulled from s = T_r d e; pushed to s = c_r d e
            for s in range(N):
                fwd_bytes[s] += res.fwd_bytes[s, rank]
                bwd_bytes[s] += res.bwd_bytes[rank, s]
            assert st["fwd_bytes_pulled"] == fwd_bytes.tolist(), (st["fwd_bytes_pulled"], fwd_bytes)
            assert st["bwd_bytes_pushed"] == bwd_bytes.tolist(), (st["bwd_bytes_pushed"], bwd_bytes)
            # ---- updated state: sigma metric on touched rows, exact elsewhere (sampled)
            c0, c1 = rank * d, (rank + 1) * d
            rows = res.U
            shard_g = ex.shard()
            gW = _np64(shard_g[torch.from_numpy(rows).to(dev)]) if rows.size else np.zeros((0, d))
            errs["W"] = max(errs["W"], assert_close(gW, shards[rank][rows], res.sigma_W[:, c0:c1], cfg.dtype,
                                                    f"iter {t} shard rows"))
            if optim == "adam" and rows.size:
                gm = _np64(ex.adam_m()[torch.from_numpy(rows).to(dev)])
                gv = _np64(ex.adam_v()[torch.from_numpy(rows).to(dev)])
                errs["m"] = max(errs["m"], assert_close(gm, m[rank][rows], res.sigma_m[:, c0:c1], cfg.dtype,
                                                        f"iter {t} adam m"))
                errs["v"] = max(errs["v"], assert_close(gv, v[rank][rows], res.sigma_v[:, c0:c1], cfg.dtype,
                                                        f"iter {t} adam v"))
            # rows outside U are bit-identical (the oracle state is resynced every iteration)
            rng = np.random.default_rng(t)
            sample = rng.integers(0, cfg.L, size=min(cfg.L, rows_sample or 4096))
            sample = np.setdiff1d(sample, rows)
            if sample.size:
                gS = _np64(shard_g[torch.from_numpy(sample).to(dev)])
                assert np.array_equal(gS, shards[rank][sample]), f"iter {t}: an untouched row changed"
            # ---- resync: the oracle continues from the GPU's (tolerance-checked) state so the next
            # forward can be compared exactly and each iteration's error is measured on its own
            _resync(shards, m, v, rank, N, rows, gW, gm if (optim == "adam" and rows.size) else None,
                    gv if (optim == "adam" and rows.size) else None)
        if report is not None:
            report.update(errs)
        return errs
    finally:
        ex.close()


def _resync(shards, m, v, rank, N, rows, gW, gm, gv):
    parts = [(rank, gW, gm, gv)]
    if N > 1:
        import torch.distributed as dist
        allp = [None] * N
        dist.all_gather_object(allp, parts[0])
        parts = allp
    for (r, w, mm, vv) in parts:
        if rows.size:
            shards[r][rows] = w
            if mm is not None:
                m[r][rows] = mm
                v[r][rows] = vv


def nonpad(ids):
    return int((np.asarray(ids) != PAD_ID).sum())
