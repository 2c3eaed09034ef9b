"""GPU-vs-oracle parity driver shared by the single-GPU tests, the co-located
multi-rank tests (N ranks of one process on one GPU), the multi-GPU torchrun
worker (tests/dist_worker.py) and __graft_entry__.smoke().

The process drives a set of LOCAL ranks: its own rank (one process per GPU,
or N = 1) or all N ranks (co-located mode, embrace.h
emb_shard_init_colocated).  It generates every rank's seeded inputs
(synthetic/), runs its ranks' part of the exchange through the C ABI, runs the
oracle for all N simulated workers on the same arrays, and compares each local
rank's outputs:
  * Y (forward output)                      exact
  * gathered ids, slot lists, counts, perm  exact (integers)
  * shard rows, Adam m / v                  sigma-normalised (tests/_metric.py);
                                            bf16 W also within 1 ulp + 2 % of the
                                            update (tests/_metric.py assert_update)
  * byte counters                           exact vs the S8 closed forms

Schedules:
  * default: flush after every iteration, compare, then resync the oracle to
    the GPU state (each iteration's error measured on its own);
  * free=True: no resync — the oracle runs free and the tolerance normaliser is
    the sigma accumulated over the iterations that touched a row
    (tests/_metric.py SigmaAcc);
  * pipelined=True (implies free): NO flush between iterations — K iterations
    back to back (the cross-iteration overlap, double buffers, side-stream
    work of the real pipeline), every Y kept, one flush at the end, then
    every Y and the final state compared.
"""

import numpy as np

from oracle import exchange, partition
from synthetic import make_workload
from synthetic.workloads import PAD_ID, gen_table

from _metric import SigmaAcc, assert_close, assert_close_acc, assert_update


def _to_torch(x, dtype, device):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype == "bf16":
        t = t.to(torch.bfloat16)          # values are already on the bf16 grid: exact
    return t.to(device)


def _np64(t):
    import torch
    return t.detach().to(torch.float64).cpu().numpy()


def make_streams(n, device):
    """n non-blocking CUDA streams for co-located ranks, created directly with
    cudaStreamCreateWithFlags (not from torch's pool, which creates dozens of
    streams at once) so that each stream gets its own hardware queue when
    CUDA_DEVICE_MAX_CONNECTIONS = 32."""
    import torch
    from cuda.bindings import runtime as rt
    torch.cuda.set_device(device)
    torch.cuda.init()
    (err,) = rt.cudaSetDevice(device)
    assert err == rt.cudaError_t.cudaSuccess, err
    out = []
    for _ in range(n):
        err, s = rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking)
        assert err == rt.cudaError_t.cudaSuccess, err
        out.append(torch.cuda.ExternalStream(int(s), device=torch.device("cuda", device)))
    _STREAMS.extend(out)            # never destroyed: a handful per test process
    return out


_STREAMS = []


class Ranks:
    """The exchange contexts this process drives and their streams."""

    def __init__(self, cfg, N, ranks, shards, device, colocated, mode, optim, lr, pad_id, max_tokens,
                 own_streams=False, table_rows=None):
        import torch
        from paper_2110_09132_b200.runtime import EmbraceExchange, make_colocated
        self.N, self.ranks, self.colocated = N, list(ranks), colocated
        dev = torch.device("cuda", device)
        kw = dict(dtype=cfg.dtype, max_tokens=max_tokens, mode=mode, optim=optim, lr=lr, pad_id=pad_id,
                  table_rows=table_rows)
        if colocated or own_streams:
            self.streams = make_streams(len(self.ranks), device)
        if colocated:
            assert self.ranks == list(range(N))
            init = [_to_torch(shards[r], cfg.dtype, dev) for r in range(N)]
            torch.cuda.synchronize()
            self.ex = make_colocated(cfg.L, cfg.D, init, self.streams, device=device, **kw)
            torch.cuda.synchronize()
            del init
        else:
            (r,) = self.ranks
            if not own_streams:
                self.streams = [torch.cuda.current_stream(dev)]
            self.ex = [EmbraceExchange(cfg.L, cfg.D, _to_torch(shards[r], cfg.dtype, dev), world=N, rank=r,
                                       device=device, **kw)]

    def items(self):
        return list(zip(self.ranks, self.ex, self.streams))

    def flush(self):
        for _, ex, s in self.items():
            ex.flush(s)

    def close(self):
        for ex in self.ex:
            ex.close()


def _gather_state(rk, rows, optim):
    """(rank, W rows, m rows, v rows) of every rank, as fp64 host arrays."""
    import torch
    out = []
    for r, ex, _ in rk.items():
        dev = ex.shard().device
        idx = torch.from_numpy(rows).to(dev)
        gW = _np64(ex.shard()[idx]) if rows.size else None
        gm = _np64(ex.adam_m()[idx]) if (optim in ("adam", "adagrad") and rows.size) else None
        gv = _np64(ex.adam_v()[idx]) if (optim == "adam" and rows.size) else None
        out.append((r, gW, gm, gv))
    if rk.N > 1 and not rk.colocated:
        import torch.distributed as dist
        allp = [None] * rk.N
        dist.all_gather_object(allp, out[0])
        out = allp
    return out


def parity_run(cfg, N=1, rank=0, mode="split", iters=3, optim=None, lr=None, pad_id=-1, last_none=True,
               device=0, rows_sample=None, ids_override=None, check=True, report=None, prefetch=False,
               colocated=False, free=False, pipelined=False, null_at=(), table_rows=None):
    """Run `iters` iterations on the local rank(s) and assert parity (see the
    module docstring for the schedules).  null_at: iterations (0-based) whose
    backward gets next_ids = NULL although more iterations follow (D_next = ∅
    mid-run: the next forward is not prefetched).  Returns the max errors."""
    import torch

    free = free or pipelined
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
    del W
    m = [np.zeros_like(s) for s in shards] if optim in ("adam", "adagrad") else None   # adagrad: accumulator
    v = [np.zeros_like(s) for s in shards] if optim == "adam" else None
    opt = exchange.OptimConfig(optim, lr=lr)
    d = cfg.D // N
    max_tokens = max(cfg.max_tokens, max(len(x) for it in wl.ids for x in it))
    ranks = list(range(N)) if colocated else [rank]
    rk = Ranks(cfg, N, ranks, shards, device, colocated, mode, optim, lr, pad_id, max_tokens, table_rows=table_rows)
    errs = {"W": 0.0, "m": 0.0, "v": 0.0, "dW_ulp": 0.0}
    fwd_bytes = {r: np.zeros(N, np.int64) for r in ranks}
    bwd_bytes = {r: np.zeros(N, np.int64) for r in ranks}
    acc = {"W": SigmaAcc(cfg.D), "m": SigmaAcc(cfg.D), "v": SigmaAcc(cfg.D)}
    keep = []          # pipelined: (k, Y per local rank, oracle Y, sigma snapshot) for the end
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    nexts = [None if ((last_none and k == iters - 1) or k in null_at) else wl.ids[k + 1] for k in range(iters)]

    def inputs(k):
        """Device inputs and outputs of iteration k for every local rank: made on
        torch's stream BEFORE any exchange call is issued (a device-wide
        synchronise while co-located ranks are mid-iteration would wait for
        gates whose peers have not been launched yet)."""
        out = {}
        for r in ranks:
            ids_t = _to_torch(wl.ids[k][r].astype(np.int32), None, dev)
            nxt_t = None if nexts[k] is None else _to_torch(nexts[k][r].astype(np.int32), None, dev)
            out[r] = (ids_t, nxt_t, _to_torch(wl.dY[k][r], cfg.dtype, dev),
                      torch.empty((len(wl.ids[k][r]), cfg.D), dtype=tdt, device=dev))
        return out

    pre = [inputs(k) for k in range(iters)] if pipelined else None
    torch.cuda.synchronize()
    try:
        for k in range(iters):
            t = k + 1
            nxt = nexts[k]
            if pipelined:
                inp = pre[k]
            else:
                inp = inputs(k)
                torch.cuda.synchronize()
            for r, ex, s in rk.items():
                ids_t, nxt_t, _, Y_t = inp[r]
                if prefetch and nxt_t is not None:
                    ex.prefetch(nxt_t, s)
                ex.forward(ids_t, Y_t, s)
            for r, ex, s in rk.items():
                ex.backward(inp[r][2], inp[r][1], s)
            Ys = {r: (inp[r][3],) for r in ranks}
            if not pipelined:
                rk.flush()
            # the rows this iteration updates (the oracle's U), before the update, for the bf16 check
            Ucat = np.unique(np.concatenate([np.asarray(x, np.int64) for x in wl.ids[k]]))
            if pad_id >= 0:
                Ucat = Ucat[Ucat != pad_id]
            old = [x[Ucat] for x in shards] if (cfg.dtype == "bf16" and not free) else None
            res = exchange.simulate_iteration(shards, wl.ids[k], wl.dY[k], nxt, t, mode, cfg.dtype, opt, m, v,
                                              pad_id)
            assert np.array_equal(res.U, Ucat)
            if not check:
                continue
            if pipelined:
                keep.append((k, {r: Ys[r][0] for r in ranks}, res.Y, acc["W"].snapshot()))
                _accumulate(acc, res, optim)
                continue
            # ---- forward: exact (free: within the sigma accumulated on the rows it reads)
            for r in ranks:
                _check_Y(Ys[r][0], res.Y[r], wl.ids[k][r], acc["W"] if free else None, cfg.dtype, f"iter {t} rank {r}")
            _check_ints(rk, wl, k, res, pad_id, t)
            for r, ex, _ in rk.items():
                st = ex.stats()
                assert st["err_flags"] == 0, f"rank {r}: device error flags {st['err_flags']}"
                # ---- byte counters (S8): pulled from s = T_r d e; pushed to s = c_r d e
                for s_ in range(N):
                    fwd_bytes[r][s_] += res.fwd_bytes[s_, r]
                    bwd_bytes[r][s_] += res.bwd_bytes[r, s_]
                assert st["fwd_bytes_pulled"] == fwd_bytes[r].tolist(), (r, st["fwd_bytes_pulled"], fwd_bytes[r])
                assert st["bwd_bytes_pushed"] == bwd_bytes[r].tolist(), (r, st["bwd_bytes_pushed"], bwd_bytes[r])
            # ---- updated state
            rows = res.U
            if free:
                _accumulate(acc, res, optim)
            state = _gather_state(rk, rows, optim)
            for (r, gW, gm, gv) in state:
                if r not in ranks or not rows.size:
                    continue
                c0, c1 = r * d, (r + 1) * d
                if free:
                    errs["W"] = max(errs["W"], assert_close_acc(gW, shards[r][rows], acc["W"].get(rows)[:, c0:c1],
                                                                cfg.dtype, f"iter {t} rank {r} shard rows (free)"))
                else:
                    errs["W"] = max(errs["W"], assert_close(gW, shards[r][rows], res.sigma_W[:, c0:c1], cfg.dtype,
                                                            f"iter {t} rank {r} shard rows"))
                    if cfg.dtype == "bf16":
                        errs["dW_ulp"] = max(errs["dW_ulp"], assert_update(gW, shards[r][rows], old[r],
                                                                           f"iter {t} rank {r} bf16 update"))
                if optim in ("adam", "adagrad"):
                    f = assert_close_acc if free else assert_close
                    sm = acc["m"].get(rows)[:, c0:c1] if free else res.sigma_m[:, c0:c1]
                    errs["m"] = max(errs["m"], f(gm, m[r][rows], sm, cfg.dtype, f"iter {t} rank {r} {optim} m"))
                if optim == "adam":
                    sv = acc["v"].get(rows)[:, c0:c1] if free else res.sigma_v[:, c0:c1]
                    errs["v"] = max(errs["v"], f(gv, v[r][rows], sv, cfg.dtype, f"iter {t} rank {r} adam v"))
            # rows outside U are bit-identical (sampled)
            rng = np.random.default_rng(t)
            sample = rng.integers(0, cfg.L, size=min(cfg.L, rows_sample or 4096))
            sample = np.setdiff1d(sample, rows)
            if free:
                sample = np.setdiff1d(sample, acc["W"].ids)
            for r, ex, _ in rk.items():
                if sample.size:
                    gS = _np64(ex.shard()[torch.from_numpy(sample).to(dev)])
                    assert np.array_equal(gS, shards[r][sample]), f"iter {t} rank {r}: an untouched row changed"
            if not free:
                # resync: the oracle continues from the GPU's (tolerance-checked) state so the next
                # forward can be compared exactly and each iteration's error is measured on its own
                for (r, gW, gm, gv) in state:
                    if rows.size:
                        shards[r][rows] = gW
                        if gm is not None:
                            m[r][rows] = gm
                        if gv is not None:
                            v[r][rows] = gv
        if pipelined and check:
            rk.flush()
            for (k, Yk, Yref, snap) in keep:
                for r in ranks:
                    _check_Y(Yk[r], Yref[r], wl.ids[k][r], snap, cfg.dtype, f"pipelined iter {k + 1} rank {r}")
            for r, ex, _ in rk.items():
                st = ex.stats()
                assert st["err_flags"] == 0, f"rank {r}: device error flags {st['err_flags']}"
            rows = acc["W"].ids
            state = _gather_state(rk, rows, optim)
            for (r, gW, gm, gv) in state:
                if r not in ranks or not rows.size:
                    continue
                c0, c1 = r * d, (r + 1) * d
                errs["W"] = max(errs["W"], assert_close_acc(gW, shards[r][rows], acc["W"].get(rows)[:, c0:c1],
                                                            cfg.dtype, f"pipelined final rank {r} shard"))
                if optim in ("adam", "adagrad"):
                    errs["m"] = max(errs["m"], assert_close_acc(gm, m[r][rows], acc["m"].get(rows)[:, c0:c1],
                                                                cfg.dtype, f"pipelined final rank {r} m"))
                if optim == "adam":
                    errs["v"] = max(errs["v"], assert_close_acc(gv, v[r][rows], acc["v"].get(rows)[:, c0:c1],
                                                                cfg.dtype, f"pipelined final rank {r} v"))
            sample = np.setdiff1d(np.random.default_rng(7).integers(0, cfg.L, size=min(cfg.L, 4096)), rows)
            for r, ex, _ in rk.items():
                if sample.size:
                    gS = _np64(ex.shard()[torch.from_numpy(sample).to(dev)])
                    assert np.array_equal(gS, shards[r][sample]), f"pipelined rank {r}: an untouched row changed"
        if report is not None:
            report.update(errs)
        return errs
    finally:
        rk.close()


def _accumulate(acc, res, optim):
    if not res.U.size:
        return
    acc["W"].add(res.U, res.sigma_W)
    if optim in ("adam", "adagrad"):
        acc["m"].add(res.U, res.sigma_m)
    if optim == "adam":
        acc["v"].add(res.U, res.sigma_v)


def _check_Y(Yt, Yref, ids, acc, dtype, what):
    gY = _np64(Yt)
    if acc is None or not acc.ids.size:
        if not np.array_equal(gY, Yref):
            bad = np.argwhere(gY != Yref)[:5]
            raise AssertionError(f"{what}: forward Y differs at {bad.tolist()}")
        return
    sig = acc.get(np.asarray(ids, np.int64))        # 0 for rows never updated: exact there
    assert_close_acc(gY, Yref, sig, dtype, f"{what}: forward Y (free)")


def _check_ints(rk, wl, k, res, pad_id, t):
    from paper_2110_09132_b200 import embrace as E
    N = rk.N
    for r, ex, _ in rk.items():
        cnts = ex.debug(E.EMB_DBG_COUNTS).reshape(N, 4)
        for n in range(N):
            ids_n = np.asarray(wl.ids[k][n], np.int64)
            assert np.array_equal(ex.debug(E.EMB_DBG_GIDS, n), ids_n), f"iter {t} rank {r}: gathered ids of {n}"
            # perm: positions sorted by (dropped, id, position); dropped = pad when pad_id >= 0
            drop = (ids_n == pad_id) if pad_id >= 0 else np.zeros(ids_n.size, bool)
            want_perm = np.lexsort((np.arange(ids_n.size), ids_n, drop))
            got_perm = ex.debug(E.EMB_DBG_PERM, n)
            if not np.array_equal(got_perm, want_perm):
                bad = np.flatnonzero(got_perm != want_perm)[:6] if got_perm.size == want_perm.size else []
                raise AssertionError(f"iter {t} rank {r}: perm of {n}: sizes {got_perm.size}/{want_perm.size}, "
                                     f"first diffs at {list(bad)}")
            want = np.concatenate([res.P_n[n], res.D_n[n]]).astype(np.int64)
            got = ex.debug(E.EMB_DBG_SLOT_IDS, n)
            assert np.array_equal(got, want), f"iter {t} rank {r}: slot ids of source {n}: {got[:8]} vs {want[:8]}"
            assert cnts[n, 0] == len(ids_n) and cnts[n, 1] == res.u[n] and cnts[n, 2] == res.p[n], \
                f"iter {t} rank {r}: counts of {n}: {cnts[n]} vs T={len(ids_n)} u={res.u[n]} p={res.p[n]}"


def graph_parity(cfg, N=1, mode="split", warm=3, nb=4, replays=2, device=0, colocated=False, rem=0,
                 graph_prefetch=False):
    """The bench's timed path: `warm` eager iterations (with emb_prefetch), one
    CUDA graph capturing a cycle of `nb` steps (forward + backward with next
    ids; `graph_prefetch`: + emb_prefetch per step, as bench.py) and emb_join,
    `replays` replays, one final eager iteration with next_ids = NULL, flush —
    then the final shard / m / v against the oracle run free over the same
    iterations.  rem > 0: bench.py's short-run path — the cycle also split
    into a graph of its first `rem` steps and one of the other nb - rem,
    replayed as: cycle, rem, rest (warm-up), `replays` cycles, rem, rest."""
    import torch
    assert nb % 2 == 0
    dev = torch.device("cuda", device)
    torch.cuda.set_device(dev)
    optim, lr = cfg.optim, cfg.lr
    W = gen_table(cfg)
    shards = partition.partition_columnwise(W, N)
    del W
    m = [np.zeros_like(s) for s in shards] if optim == "adam" else None
    v = [np.zeros_like(s) for s in shards] if optim == "adam" else None
    wl = make_workload(cfg, N, nb)
    ranks = list(range(N)) if colocated else [0]
    rk = Ranks(cfg, N, ranks, shards, device, colocated, mode, optim, lr, -1, cfg.max_tokens, own_streams=True)
    ids_d = {r: [_to_torch(wl.ids[b][r].astype(np.int32), None, dev) for b in range(nb)] for r in ranks}
    dY_d = {r: [_to_torch(wl.dY[b][r], cfg.dtype, dev) for b in range(nb)] for r in ranks}
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    Y_d = {r: [torch.empty((len(wl.ids[b][r]), cfg.D), dtype=tdt, device=dev) for b in range(nb)] for r in ranks}
    torch.cuda.synchronize()
    from paper_2110_09132_b200 import embrace as E
    seq = []                       # batch index of every executed iteration, in order
    try:
        for k in range(warm):
            b = k % nb
            for r, ex, s in rk.items():
                ex.prefetch(ids_d[r][(b + 1) % nb], s)
                ex.forward(ids_d[r][b], Y_d[r][b], s)
            for r, ex, s in rk.items():
                ex.backward(dY_d[r][b], ids_d[r][(b + 1) % nb], s)
            seq.append(b)
        for r, ex, s in rk.items():
            E.emb_join(ex.ctx, s)
        torch.cuda.synchronize()
        def capture(j0, n):
            out = []
            for r, ex, s in rk.items():
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for j in range(j0, j0 + n):
                        b = (warm + j) % nb
                        if graph_prefetch:
                            E.emb_prefetch(ex.ctx, ids_d[r][(b + 1) % nb], s)
                        E.emb_forward_exchange(ex.ctx, ids_d[r][b], Y_d[r][b], s)
                        E.emb_backward_exchange(ex.ctx, dY_d[r][b], ids_d[r][(b + 1) % nb], s)
                    E.emb_join(ex.ctx, s)
                out.append((g, s))
            return out

        def replay(gs, j0, n):
            for g, s in gs:
                with torch.cuda.stream(s):      # replay() launches on the CURRENT stream
                    g.replay()
            seq.extend((warm + j) % nb for j in range(j0, j0 + n))

        graphs = capture(0, nb)
        if rem:
            g_rem, g_comp = capture(0, rem), capture(rem, nb - rem)
        torch.cuda.synchronize()
        if rem:
            replay(graphs, 0, nb)
            replay(g_rem, 0, rem)
            replay(g_comp, rem, nb - rem)
        for _ in range(replays):
            replay(graphs, 0, nb)
        if rem:
            replay(g_rem, 0, rem)
            replay(g_comp, rem, nb - rem)
        b = (warm + replays * nb) % nb
        for r, ex, s in rk.items():
            ex.forward(ids_d[r][b], Y_d[r][b], s)
        for r, ex, s in rk.items():
            ex.backward(dY_d[r][b], None, s)
        seq.append(b)
        rk.flush()
        # oracle, free-running over the executed sequence
        acc = {"W": SigmaAcc(cfg.D), "m": SigmaAcc(cfg.D), "v": SigmaAcc(cfg.D)}
        opt = exchange.OptimConfig(optim, lr=lr)
        for i, b in enumerate(seq):
            nxt = wl.ids[seq[i + 1]] if i + 1 < len(seq) else None
            snap = acc["W"].snapshot()
            res = exchange.simulate_iteration(shards, wl.ids[b], wl.dY[b], nxt, i + 1, mode, cfg.dtype, opt, m, v)
            _accumulate(acc, res, optim)
            if i == len(seq) - 1:
                for r in ranks:
                    _check_Y(Y_d[r][b], res.Y[r], wl.ids[b][r], snap, cfg.dtype, f"graph path, last forward rank {r}")
        for r, ex, _ in rk.items():
            assert ex.stats()["err_flags"] == 0
        rows = acc["W"].ids
        d = cfg.D // N
        errs = {}
        for (r, gW, gm, gv) in _gather_state(rk, rows, optim):
            c0, c1 = r * d, (r + 1) * d
            errs[f"W{r}"] = assert_close_acc(gW, shards[r][rows], acc["W"].get(rows)[:, c0:c1], cfg.dtype,
                                             f"graph path rank {r} shard")
            if optim == "adam":
                assert_close_acc(gm, m[r][rows], acc["m"].get(rows)[:, c0:c1], cfg.dtype, f"graph path rank {r} m")
                assert_close_acc(gv, v[r][rows], acc["v"].get(rows)[:, c0:c1], cfg.dtype, f"graph path rank {r} v")
        return errs, len(seq)
    finally:
        rk.close()


def nonpad(ids):
    return int((np.asarray(ids) != PAD_ID).sum())
