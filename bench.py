#!/usr/bin/env python
"""bench.py — EmbRace sparse-embedding fwd+bwd exchange throughput on B200.

One step = emb_forward_exchange + emb_backward_exchange of one synthetic batch
per rank (all of SURVEY §8(a): id all-gather, pull-gather forward, next-id
prefetch + D_next marks, per-source sort/unique/split, sender coalesce + push,
owner merge + fused optimizer update, scheduled part on the side stream).  The
timed region ends after every deferred (scheduled) update has completed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config lstm_lm]
                  [--mode split] [--impl ours|reference] [--no-graph]

N > 1 runs under torchrun (one process per GPU).  Default workload:
BASELINE.json configs[1] (LSTM-LM 793,470 x 512 fp32, 128 x 35 Zipf batches per
rank, SPLIT mode, Adam) — the configuration the metric is quoted on; it fits
one GPU.  Prints ONE JSON line on rank 0.
"""

import argparse
import json
import os
import statistics
import sys
import threading
import time

# The CPU baseline (the oracle) is single-threaded by construction: the thread
# pools of every BLAS NumPy may link are pinned to one thread BEFORE NumPy is
# imported (setting them later has no effect), and cpu_baseline() pins the
# process to one core while it runs.
for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMEXPR_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synthetic import get_config  # noqa: E402
from synthetic.workloads import PAD_ID, gen_dY, gen_ids, gen_table  # noqa: E402

L2_BYTES = 126 * 1024 * 1024
METRIC = "sparse embedding fwd+bwd exchange tokens/s at 1/2/4/8 B200; % HBM/NVLink roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="lstm_lm")
    ap.add_argument("--mode", default="split", choices=["raw", "coal", "split"])
    ap.add_argument("--baseline", default=None, choices=["allgather", "allreduce"],
                    help="NEXT-2: time an in-box baseline (baselines/inbox.py) instead of the exchange")
    ap.add_argument("--schedule", action="store_true",
                    help="NEXT-1: Computation Stall of FIFO / Horizontal / 2D scheduling (separate JSON line)")
    ap.add_argument("--batch-mult", type=int, default=1,
                    help="tokens per rank x M (sequences per rank, or max tokens when packed): the bandwidth-"
                         "regime sweep of SURVEY §7 (cap 32768 tokens per rank)")
    ap.add_argument("--tables", type=int, default=1, choices=[1, 2],
                    help="NEXT-3: exchange this many stacked tables (same shape) in one call")
    ap.add_argument("--optim", default=None, choices=["sgd", "adam", "adagrad"],
                    help="override the config's sparse optimizer (NEXT-4: adagrad)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--graph-no-prefetch", action="store_true",
                    help="capture the graph without emb_prefetch (round-1 timed path)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=64)
    ap.add_argument("--dense-queue", type=int, default=0, metavar="W",
                    help="measure the a13 dense AllReduce priority queue with window W (separate JSON line)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------- clocks (NVML, sampled in a thread)
class ClockSampler:
    def __init__(self, device_index, period_s=0.002):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.period = period_s
        self.ok = False
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- NVLink traffic (NVML counters)
def nvlink_kib(local):
    """Cumulative NVLink data KiB (TX, RX) of this rank's GPU over all links
    (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX), or None."""
    try:
        import pynvml as nv
        import torch
        nv.nvmlInit()
        try:
            pr = torch.cuda.get_device_properties(local)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            h = nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            h = nv.nvmlDeviceGetHandleByIndex(local)
        vals = nv.nvmlDeviceGetFieldValues(h, [nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                               nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX])
        if any(v.nvmlReturn != 0 for v in vals):
            return None
        return [int(v.value.ullVal) for v in vals]
    except Exception:
        return None


# ---------------------------------------------------------------- workload
def n_batches(cfg, N):
    """Enough distinct batches that the inputs+outputs cycled through exceed
    2x L2 (126 MB) between reuse (timing rule: inputs larger than L2)."""
    esz = 2 if cfg.dtype == "bf16" else 4
    per = 2 * cfg.max_tokens * cfg.D * esz           # dY read + Y written per batch
    nb = int(np.ceil(2 * L2_BYTES / per))
    nb += nb % 2                                     # even: graph replays keep the parity
    return max(4, min(nb, 64))


def traffic_for(config, world, kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the newest committed
    ncu --set full capture (profiles/*traffic.json), or None if not captured."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*traffic.json")))
    if not files:
        return None
    d = json.load(open(files[-1])).get(f"{config}/n{world}", {})
    return d.get(kernel)


def algorithmic_bytes(cfg, N, rank, ids_all, next_all, mode):
    """Per-kernel algorithmic bytes of one step on `rank`,
    from the actual ids.  Returns {kernel: (hbm_bytes, nvlink_bytes)}."""
    esz = 2 if cfg.dtype == "bf16" else 4
    d = cfg.D // N
    T = [len(x) for x in ids_all]
    ids_r = np.asarray(ids_all[rank])
    u_fwd = len(np.unique(ids_r))
    U_n = [np.unique(x) for x in ids_all]
    u = [len(x) for x in U_n]
    Uall = np.unique(np.concatenate(ids_all))
    nxt = np.unique(np.concatenate(next_all))
    P = np.intersect1d(Uall, nxt).size if mode == "split" else Uall.size
    Q = Uall.size - P
    out = {}
    # forward: Y write + distinct rows read (every owner's slice) + ids; NVLink in: every distinct row's
    # N-1 remote slices once (the volume a deduplicating pull must move; the paper's plain AlltoAll
    # moves (N-1)*T*d*e, reading R10)
    out["fwd_pull_gather"] = (T[rank] * cfg.D * esz + u_fwd * cfg.D * esz + T[rank] * 4,
                              (N - 1) * u_fwd * d * esz)
    # a5 prefetch push (+ D_next marks in SPLIT); a6 sort (aux stream); a8 tables (aux)
    out["mark_next"] = (T[rank] * 4 * (N + 1) + (sum(T) * 8 if mode == "split" else 0), (N - 1) * T[rank] * 4)
    out["sort_unique"] = (sum(T) * 4 * 3 + sum(u) * 4 * 4 + (sum(u) * 8 if N > 1 else 0), 0)
    out["split_tables"] = (sum(u) * 4 * 3, 0)
    opt_b = {"adam": 16, "adagrad": 8}.get(cfg.optim, 0)   # Adam m, v / Adagrad accumulator, fp32: read + write
    row_state = 2 * esz + opt_b               # shard row element read + write (+ m, v)
    if mode == "raw":
        out["rawpush"] = (T[rank] * cfg.D * esz * 2, (N - 1) * T[rank] * d * esz)
        out["rawcoal"] = (sum(T) * d * esz + sum(u) * d * 4, 0)
        src = 4
    elif N == 1:
        # a7: dY read once; a11: the optimizer step applied by coal_apply (no exchange, no merge)
        out["coal_push"] = (T[rank] * cfg.D * esz, 0)
        out["coal_apply"] = (Uall.size * cfg.D * row_state, 0)
        return out
    else:
        c_r = u[rank]
        out["coal_push"] = (T[rank] * cfg.D * esz, 0)
        # a9/a10: the coalesced rows land in the owners' receive rows (or the stage)
        out["coal_apply"] = (c_r * cfg.D * esz, (N - 1) * c_r * d * esz)
        src = esz
    frac_p = (P / Uall.size) if Uall.size else 0
    contrib = sum(u) * d * src
    out["merge_update_prior"] = (int(frac_p * contrib) + P * d * row_state, 0)
    if mode == "split":
        q_r = len(np.setdiff1d(U_n[rank], nxt))
        out["defpush"] = (2 * q_r * cfg.D * esz, (N - 1) * q_r * d * esz)
        out["merge_update_sched"] = (int((1 - frac_p) * contrib) + Q * d * row_state, 0)
    return out


# ---------------------------------------------------------------- several tables in one exchange (NEXT-3)
# --tables 2: the config's table twice, stacked row-wise (embrace.h num_tables):
# table A looked up by the batch's tokens, table B by a second token stream of
# the same shape (LM: input and softmax tables; GNMT: encoder and decoder), B's
# ids offset by L (global row ids).  One forward + backward serves both.
TABLES = 1
BASE_CFG = None
PADS = {PAD_ID}


def stacked(cfg, tables):
    """(sizing config, per-table row counts): L and max_tokens of the stacked exchange."""
    global TABLES, BASE_CFG, PADS
    TABLES, BASE_CFG = tables, cfg
    if tables == 1:
        return cfg, None
    import dataclasses
    PADS = {PAD_ID + k * cfg.L for k in range(tables)}
    big = dataclasses.replace(cfg, L=cfg.L * tables, **({"seq_len": cfg.seq_len * tables} if cfg.packed
                                                        else {"batch": cfg.batch * tables}))
    return big, [cfg.L] * tables


def gen_ids_t(cfg, b, r):
    if TABLES == 1:
        return gen_ids(cfg, b, r)
    c0 = BASE_CFG
    return np.concatenate([k * c0.L + gen_ids(c0, b + 7919 * k, r) for k in range(TABLES)]).astype(np.int32)


def gen_table_t(cfg):
    if TABLES == 1:
        return gen_table(cfg)
    W = gen_table(BASE_CFG)
    return np.vstack([W] * TABLES)


def count_nonpad(x):
    x = np.asarray(x)
    return int(sum(int((x != pid).sum()) for pid in PADS) - (len(PADS) - 1) * x.size)


def make_batches(cfg, N, rank, nb):
    ids = [gen_ids_t(cfg, b, rank) for b in range(nb)]
    ids_all = [[gen_ids_t(cfg, b, s) for s in range(N)] for b in range(nb)] if N > 1 else [[x] for x in ids]
    dY = [gen_dY(cfg, b, rank, len(ids[b])) for b in range(nb)]
    return ids, ids_all, dY


# ---------------------------------------------------------------- oracle timing (CPU baseline / reference arm)
def oracle_step_fn(cfg, N, mode, budget_s):
    """Returns (step(k) -> tokens processed, sample description).  The oracle
    simulates all N workers of one iteration of the same workload; if a full
    iteration exceeds `budget_s`, each step runs on the first B' sequences of
    every rank (a bounded sample) and counts only those tokens."""
    from oracle import exchange, partition
    opt = exchange.OptimConfig(cfg.optim, lr=cfg.lr)
    W = gen_table_t(cfg)
    shards = partition.partition_columnwise(W, N)
    del W
    m = [np.zeros_like(s) for s in shards] if cfg.optim in ("adam", "adagrad") else None
    v = [np.zeros_like(s) for s in shards] if cfg.optim == "adam" else None
    nb = 4
    ids = [[gen_ids_t(cfg, b, s) for s in range(N)] for b in range(nb)]
    dY = [[gen_dY(cfg, b, s, len(ids[b][s])) for s in range(N)] for b in range(nb)]
    state = {"t": 0, "frac": 1.0}

    def run(k, frac):
        b = k % nb
        cut = [max(1, int(len(x) * frac)) for x in ids[b]]
        I = [ids[b][s][: cut[s]] for s in range(N)]
        G = [dY[b][s][: cut[s]] for s in range(N)]
        nxt = [ids[(b + 1) % nb][s][: cut[s]] for s in range(N)]
        state["t"] += 1
        exchange.simulate_iteration(shards, I, G, nxt, state["t"], mode, cfg.dtype, opt, m, v)
        return sum(count_nonpad(x) for x in I)

    t0 = time.perf_counter()
    run(0, 1.0)
    full = time.perf_counter() - t0
    if full > budget_s:
        state["frac"] = max(0.02, budget_s / full)
    frac = state["frac"]
    desc = (f"oracle.exchange.simulate_iteration, {N} simulated worker(s), mode {mode}; "
            + ("full iterations" if frac >= 1.0 else f"first {frac:.1%} of every rank's batch per step"))
    return (lambda k: run(k, frac)), desc


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


class pinned_core:
    """Pin this process to one core (the lowest it may run on) for the block."""

    def __enter__(self):
        self.old = os.sched_getaffinity(0)
        self.core = min(self.old)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *a):
        os.sched_setaffinity(0, self.old)


def host_info(pin):
    return {"cores": 1, "pinned_core": pin.core, "host_cpu_count": os.cpu_count(), "cpu_model": cpu_model(),
            "threads_env": {v: os.environ.get(v) for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS",
                                                              "MKL_NUM_THREADS")}}


def cpu_baseline(cfg, N, mode, seconds=12.0):
    with pinned_core() as pin:
        step, desc = oracle_step_fn(cfg, N, mode, budget_s=seconds / 3)
        toks, k = 0, 1
        t0 = time.perf_counter()
        while True:
            toks += step(k)
            k += 1
            el = time.perf_counter() - t0
            if el > seconds or k > 200:
                break
    out = {"value": toks / el, "unit": "tokens/s", "kind": "oracle",
           "sample": f"{desc}; {k - 1} timed steps in {el:.1f} s (single-threaded NumPy, pinned to one core)"}
    out.update(host_info(pin))
    return out


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return
    with pinned_core() as pin:
        step, desc = oracle_step_fn(cfg, world, args.mode, budget_s=1.0)
        for k in range(args.warmup):
            step(k)
        toks = 0
        t0 = time.perf_counter()
        for k in range(args.steps):
            toks += step(args.warmup + k)
        el = time.perf_counter() - t0
    val = toks / el
    cpu = {"value": val, "unit": "tokens/s", "kind": "oracle", "sample": desc}
    cpu.update(host_info(pin))
    line = {"metric": METRIC, "value": val, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name} (oracle on host cores)", "mode": args.mode, "ranks": world},
            "impl": "reference",
            "cpu_baseline": cpu,
            "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- a13 dense queue (separate measurement)
def run_dense(args, cfg, world, rank, local):
    """the dense queue is measured separately and in a concurrent
    run for interference; it is not part of the headline.  Per iteration every
    rank enqueues the config's dense blocks in BP order (last layer first) with
    priority = FP order (block 0 = first layer = most urgent),
    window W (reading R16), then flushes.  Three timed phases (CUDA events on
    the launching stream, max over ranks): queue alone, sparse step alone
    (eager), both concurrently (the queue's comm stream overlaps the next
    iterations' sparse exchange)."""
    import torch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_2110_09132_b200 import embrace as E
    from paper_2110_09132_b200.runtime import EmbraceExchange
    from synthetic.workloads import gen_dense

    nblk = cfg.dense_blocks or 16
    nel = cfg.dense_block_elems or 8_400_000
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    blocks = [torch.from_numpy(gen_dense(cfg, k, rank, 1 << 16)).to(tdt).to(dev).repeat((nel >> 16) + 1)[:nel]
              .contiguous() for k in range(nblk)]
    nb = n_batches(cfg, world)
    ids, ids_all, dY = make_batches(cfg, world, rank, nb)
    ids_d = [torch.from_numpy(x).to(dev) for x in ids]
    dY_d = [torch.from_numpy(x).to(dev).to(tdt) for x in dY]
    Y_d = [torch.empty((len(x), cfg.D), dtype=tdt, device=dev) for x in ids]
    d = cfg.D // world
    W = gen_table(cfg)
    shard0 = torch.from_numpy(np.ascontiguousarray(W[:, rank * d:(rank + 1) * d])).to(dev).to(tdt)
    del W
    ex = EmbraceExchange(cfg.L, cfg.D, shard0, world=world, rank=rank, device=local, dtype=cfg.dtype,
                         max_tokens=cfg.max_tokens, mode=args.mode, optim=cfg.optim, lr=cfg.lr,
                         dense_queue=True, queue_window=args.dense_queue)
    stream = torch.cuda.current_stream()
    ready = torch.cuda.Event()
    prios = list(range(nblk))[::-1]          # enqueued in BP order: the last layer (largest FP index) first
    last = []

    seq = [0]  # global step counter: the batch sequence continues across the timed phases (each forward
               # must see the ids the previous backward promised)

    def sparse(_k):
        b = seq[0] % nb
        seq[0] += 1
        E.emb_prefetch(ex.ctx, ids_d[(b + 1) % nb], stream)
        E.emb_forward_exchange(ex.ctx, ids_d[b], Y_d[b], stream)
        E.emb_backward_exchange(ex.ctx, dY_d[b], ids_d[(b + 1) % nb], stream)

    def dense():
        ready.record(stream)                 # the blocks' BP is done (stand-in: everything so far on `stream`)
        tk = [E.dense_allreduce_enqueue(ex.ctx, blocks[p], p, ready) for p in prios]
        E.dense_queue_flush(ex.ctx)          # issued before `ready` is re-recorded (borrowed event)
        last[:] = tk

    def timed(fn, K):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        last.clear()
        fn(K)
        E.emb_join(ex.ctx, stream)           # deferred sparse parts
        for tk in last:                      # the queue's comm stream (in-order: the last iteration suffices)
            E.dense_wait(ex.ctx, tk, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([ms], device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            ms = float(tt.item())
        return ms

    def q_only(K):
        for _ in range(K):
            dense()

    def s_only(K):
        for j in range(K):
            sparse(j)

    def both(K):
        for j in range(K):
            sparse(j)
            dense()

    K = max(3, min(args.steps, 50))
    for fn in (q_only, s_only, both):       # warm-up (NCCL communicator, kernels)
        timed(fn, max(3, args.warmup // 4))
    with ClockSampler(local) as clk:
        t_q = timed(q_only, K)
        t_s = timed(s_only, K)
        t_b = timed(both, K)
    log = [int(x) for x in ex.debug(E.EMB_DBG_ISSUE_LOG)]
    want1 = [int(x) for x in E.emb_queue_issue_order(prios, args.dense_queue)]
    per_iter = [x % nblk for x in log[:nblk]]
    order_ok = per_iter == want1
    bytes_blk = nel * (2 if cfg.dtype == "bf16" else 4)
    tot = nblk * bytes_blk
    busbw = (2 * (world - 1) / world * tot) / (t_q / K * 1e-3) / 1e9 if world > 1 else 0.0
    algbw = tot / (t_q / K * 1e-3) / 1e9
    nvl_peak = 770.0
    ex.flush()
    if rank == 0:
        line = {"metric": "dense AllReduce priority queue (a13): bus GB/s per rank", "value": round(busbw, 1),
                "unit": "GB/s", "n_gpus": world, "steps": K, "warmup": max(3, args.warmup // 4),
                "ms_per_step": t_q / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": cfg.dtype, "data": "synthetic",
                "config": {"workload": f"{cfg.name}: {nblk} dense blocks x {nel} {cfg.dtype} per rank "
                                       f"({tot / 2**20:.0f} MiB), priority = FP order, enqueued in BP order",
                           "window": args.dense_queue, "sparse_mode": args.mode},
                "algbw_gbs": round(algbw, 1),
                "roofline": {"bound": "nvlink", "achieved": round(busbw, 1), "peak": nvl_peak, "unit": "GB/s",
                             "frac": round(busbw / nvl_peak, 4) if world > 1 else None,
                             "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s/direction; ring "
                                            "bus bytes 2(N-1)/N x buffer (NVLS may exceed it)"},
                "issue_order": {"first_iteration": per_iter, "rule": want1, "ok": order_ok},
                "interference": {"queue_ms": t_q / K, "sparse_ms": t_s / K, "both_ms": t_b / K,
                                 "overlap_frac": round((t_q + t_s - t_b) / min(t_q, t_s), 4)
                                 if min(t_q, t_s) > 0 else None,
                                 "note": "sparse steps eager (no graph); overlap_frac 1 = the shorter phase "
                                         "is fully hidden"},
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    ex.close()
    if world > 1:
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------- NEXT-1: 2D schedule and Computation Stall
def run_schedule(args, cfg, world, rank, local):
    """SURVEY §8(f) NEXT-1 (PAPER.md:282-336 Horizontal / Vertical / 2D
    Scheduling, PAPER.md:542-550 Computation Stall).  A synthetic training step
    around the real exchange: embedding FP (emb_forward_exchange), K dense
    blocks' FP (GEMM stand-ins, block k = one [T, H] x [H, H] bf16 GEMM of the
    config's dense-block size), their BP in reverse (two GEMMs each; the weight
    gradient's AllReduce enqueued into the a13 priority queue as soon as it is
    produced, priority = FP order), embedding BP (emb_backward_exchange).  The
    FP of block k of the next iteration consumes block k's averaged gradient.
      fifo        Default Scheduling: queue window 1 (issue in BP order), COAL
                  exchange, and the next FP waits for EVERY AllReduce
                  (PAPER.md:323-325);
      horizontal  priority queue (window = K: issued at the end of BP in FP
                  order), the next iteration's embedding FP first, block k's FP
                  waits only for block k's AllReduce; COAL;
      2d          horizontal + Vertical Scheduling (SPLIT: only the prior part
                  precedes the next FP, the deferred part on the lowest-priority
                  side stream).
    Computation Stall = step time - compute-only step time (the same GEMMs, no
    exchange, no AllReduce): the GPU idle time plus, for 2d, the Vertical
    Scheduling computation.  Device time on the main stream,
    CUDA events, max over ranks."""
    import torch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_2110_09132_b200 import embrace as E
    from paper_2110_09132_b200.runtime import EmbraceExchange

    K = cfg.dense_blocks or 16
    H = 2048
    H2 = max(256, (cfg.dense_block_elems or 8_400_000) // H // 128 * 128)  # block weight [H, H2] ~ the config's size
    nb = 4
    ids, ids_all, dY = make_batches(cfg, world, rank, nb)
    T = min(len(x) for x in ids)
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    ids_d = [torch.from_numpy(x).to(dev) for x in ids]
    dY_d = [torch.from_numpy(x).to(dev).to(tdt) for x in dY]
    Y_d = [torch.empty((len(x), cfg.D), dtype=tdt, device=dev) for x in ids]
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    Wb = [torch.randn(H, H2, device=dev, dtype=torch.bfloat16, generator=g) * 0.01 for _ in range(K)]
    Wb2 = [torch.randn(H2, H, device=dev, dtype=torch.bfloat16, generator=g) * 0.01 for _ in range(K)]
    Gb = [torch.zeros(H, H2, device=dev, dtype=torch.bfloat16) for _ in range(K)]
    stream = torch.cuda.current_stream()
    d = cfg.D // world
    Wt = gen_table_t(cfg)
    shard0 = torch.from_numpy(np.ascontiguousarray(Wt[:, rank * d:(rank + 1) * d])).to(dev).to(tdt)
    del Wt

    def x_from(Y):  # the blocks' input: the embedding rows (width D) tiled / cut to H
        x = Y[:T].to(torch.bfloat16)
        return x.repeat(1, (H + cfg.D - 1) // cfg.D)[:, :H].contiguous()

    def step_compute(k, ex, sched, tickets):
        b = k % nb
        nxt = ids_d[(b + 1) % nb]
        if ex is not None:
            if sched.startswith("fifo"):
                for tk in tickets:                       # Default: every AllReduce before the next FP
                    E.dense_wait(ex.ctx, tk, stream)
            E.emb_prefetch(ex.ctx, nxt, stream)
            E.emb_forward_exchange(ex.ctx, ids_d[b], Y_d[b], stream)   # embedding FP first
            x = x_from(Y_d[b])
        else:
            x = x_from(Y_d[b])
        acts = []
        for j in range(K):                                # dense FP, block j needs its averaged gradient
            if ex is not None and not sched.startswith("fifo") and tickets:
                E.dense_wait(ex.ctx, tickets[j], stream)
            acts.append(x)
            x = torch.relu(x @ Wb[j]) @ Wb2[j]
        dx = x
        ready = []
        new_tickets = [None] * K
        for j in reversed(range(K)):                      # dense BP: weight grad, then its AllReduce
            h = torch.relu(acts[j] @ Wb[j])
            dh = dx @ Wb2[j].t()
            torch.matmul(acts[j].t(), dh, out=Gb[j])
            dx = dh @ Wb[j].t()
            if ex is not None:
                ev = torch.cuda.Event()
                ev.record(stream)
                ready.append(ev)                          # borrowed by the queue until issued
                new_tickets[j] = E.dense_allreduce_enqueue(ex.ctx, Gb[j], j, ev)
            del h
        if ex is not None:
            E.emb_backward_exchange(ex.ctx, dY_d[b], nxt, stream)   # embedding BP (sparse exchange)
            E.dense_queue_flush(ex.ctx)
        return new_tickets, ready

    def timed(ex, sched, iters, warm):
        tickets, keep = [], []
        for k in range(warm):
            tickets, r = step_compute(k, ex, sched, tickets)
            keep.append(r)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(warm, warm + iters):
            tickets, r = step_compute(k, ex, sched, tickets)
            keep.append(r)
        if ex is not None:
            for tk in tickets:
                E.dense_wait(ex.ctx, tk, stream)
            E.emb_join(ex.ctx, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        if world > 1:
            tt = torch.tensor([ms], device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            ms = float(tt.item())
        return ms * 1e3

    iters, warm = max(5, min(args.steps, 30)), max(3, min(args.warmup, 5))
    compute_us = timed(None, None, iters, warm)
    res = {}
    # the deterministic window rule (reading R16) stands in for the paper's
    # ready-based priority pop: W = how many ready blocks may wait behind the
    # comm stream; W = K holds everything until the end of BP (FP order)
    for sched, mode, window in (("fifo", "coal", 1), ("horizontal_w2", "coal", 2), ("horizontal_w4", "coal", 4),
                                ("horizontal", "coal", K), ("2d_w4", "split", 4), ("2d", "split", K)):
        ex = EmbraceExchange(cfg.L, cfg.D, shard0, world=world, rank=rank, device=local, dtype=cfg.dtype,
                             max_tokens=cfg.max_tokens, mode=mode, optim=cfg.optim, lr=cfg.lr, dense_queue=True,
                             queue_window=window)
        step_us = timed(ex, sched, iters, warm)
        ex.flush()
        ex.close()
        res[sched] = {"step_us": round(step_us, 1), "stall_us": round(step_us - compute_us, 1),
                      "sparse_mode": mode, "queue_window": window}
    if rank == 0:
        line = {"metric": "2D-schedule computation stall (NEXT-1): step time - compute-only time",
                "value": min(res["2d"]["stall_us"], res["2d_w4"]["stall_us"]), "unit": "us per iteration", "n_gpus": world, "steps": iters,
                "warmup": warm, "higher_is_better": False, "dtype": cfg.dtype, "data": "synthetic",
                "config": {"workload": f"{cfg.name}: embedding exchange + {K} dense blocks "
                                       f"([{T}, {H}] x [{H}, {H2}] bf16 GEMM pairs), per-block AllReduce "
                                       f"{H * H2 * 2 / 2**20:.1f} MiB bf16"},
                "compute_only_us": round(compute_us, 1), "schedules": res,
                "stall_ratio_fifo_over_2d": round(res["fifo"]["stall_us"] / res["2d"]["stall_us"], 3)
                if res["2d"]["stall_us"] > 0 else None}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------- NEXT-2: in-box baselines
def run_baseline(args, cfg, world, rank, local):
    """the same workload through baselines/inbox.py
    (Horovod-AllGather-style sparse aggregation or dense-gradient AllReduce, a
    replicated table per rank, torch ops + NCCL), timed like the main arm
    (CUDA events, max over ranks; eager: the collectives' sizes are host-side).
    One JSON line, impl "inbox_<kind>"; compare with the main arm's value."""
    import torch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from baselines.inbox import ReplicatedTable
    nb = n_batches(cfg, world)
    ids, ids_all, dY = make_batches(cfg, world, rank, nb)
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    ids_d = [torch.from_numpy(x.astype(np.int64)).to(dev) for x in ids]
    dY_d = [torch.from_numpy(x).to(dev).to(tdt) for x in dY]
    W = torch.from_numpy(gen_table_t(cfg)).to(dev).to(tdt)
    rt = ReplicatedTable(W, optim=cfg.optim, lr=cfg.lr, world=world, kind=args.baseline)
    del W
    stream = torch.cuda.current_stream()

    def step(k):
        b = k % nb
        rt.forward(ids_d[b])
        rt.backward(ids_d[b], dY_d[b], cfg.max_tokens)

    for k in range(args.warmup):
        step(k)
    K = min(args.steps, 200)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for j in range(K):
            step(args.warmup + j)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    tok = sum(count_nonpad(ids_all[(args.warmup + j) % nb][s]) for j in range(K) for s in range(world))
    esz = 2 if cfg.dtype == "bf16" else 4
    wire = ((world - 1) * cfg.max_tokens * (cfg.D * esz + 8) if args.baseline == "allgather"
            else 2 * (world - 1) / world * cfg.L * cfg.D * 4) if world > 1 else 0
    if rank == 0:
        line = {"metric": METRIC, "value": tok / (ms / 1e3), "unit": "tokens/s", "n_gpus": world, "steps": K,
                "warmup": args.warmup, "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": {"fp32": "f32", "bf16": "bf16"}[cfg.dtype], "data": "synthetic",
                "impl": f"inbox_{args.baseline}",
                "config": {"workload": f"{cfg.name}: L={cfg.L} D={cfg.D} {cfg.dtype}, replicated table per rank",
                           "aggregation": {"allgather": "all_gather_into_tensor of every rank's padded (ids, dY) "
                                                        "+ local coalesce (Horovod AllGather)",
                                           "allreduce": "dense [L, D] fp32 gradient AllReduce (Horovod dense)"}
                           [args.baseline], "optim": cfg.optim},
                "wire_bytes_per_rank_per_step": int(wire), "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    world, rank, local = dist_env()
    if world != args.gpus:
        world = args.gpus if world == 1 else world
    cfg = get_config(args.config)
    if args.batch_mult > 1:
        import dataclasses
        cfg = dataclasses.replace(cfg, **({"seq_len": cfg.seq_len * args.batch_mult} if cfg.packed
                                          else {"batch": cfg.batch * args.batch_mult}))
    if args.optim:
        import dataclasses
        cfg = dataclasses.replace(cfg, optim=args.optim, lr=cfg.lr if args.optim == "adam" else 1e-2)
    cfg, table_rows = stacked(cfg, args.tables)
    if args.impl == "reference":
        return run_reference(args, cfg, world, rank)
    if args.dense_queue:
        return run_dense(args, cfg, world, rank, local)
    if args.schedule:
        return run_schedule(args, cfg, world, rank, local)
    if args.baseline:
        return run_baseline(args, cfg, world, rank, local)

    import torch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_2110_09132_b200 import embrace as E
    from paper_2110_09132_b200.runtime import EmbraceExchange

    mode = args.mode
    nb = n_batches(cfg, world)
    ids, ids_all, dY = make_batches(cfg, world, rank, nb)
    ids_d = [torch.from_numpy(x).to(dev) for x in ids]
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    dY_d = [torch.from_numpy(x).to(dev).to(tdt) for x in dY]
    Y_d = [torch.empty((len(x), cfg.D), dtype=tdt, device=dev) for x in ids]
    d = cfg.D // world
    W = gen_table_t(cfg)
    shard0 = torch.from_numpy(np.ascontiguousarray(W[:, rank * d:(rank + 1) * d])).to(dev).to(tdt)
    del W
    ex = EmbraceExchange(cfg.L, cfg.D, shard0, world=world, rank=rank, device=local, dtype=cfg.dtype,
                         max_tokens=cfg.max_tokens, mode=mode, optim=cfg.optim, lr=cfg.lr,
                         timeout_ms=int(os.environ.get("EMB_TIMEOUT_MS", "10000")), table_rows=table_rows)
    del shard0
    stream = torch.cuda.current_stream()

    def step(k):
        b = k % nb
        # the paper's prefetch: the next batch's ids are in memory before this
        # step starts; emb_prefetch lets its work overlap the forward
        E.emb_prefetch(ex.ctx, ids_d[(b + 1) % nb], stream)
        E.emb_forward_exchange(ex.ctx, ids_d[b], Y_d[b], stream)
        E.emb_backward_exchange(ex.ctx, dY_d[b], ids_d[(b + 1) % nb], stream)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    _align = torch.zeros(1, device=dev)

    def device_align():
        # N > 1: a one-element NCCL all_reduce on `stream` right before the start event, so that the
        # ranks' timed regions start together on the device (the host barrier alone leaves the ranks'
        # first launches up to ~0.3 ms apart, which a short run would count as exchange time)
        if world > 1:
            torch.distributed.all_reduce(_align)

    def check_err(phase):  # sticky device error bits (1 id range, 2 state, 4 peer-wait timeout)
        torch.cuda.synchronize()
        ef = ex.stats()["err_flags"]
        if ef:
            info = E.emb_debug_copy(ex.ctx, E.EMB_DBG_ERRINFO).reshape(8, 4)
            waits = [tuple(int(v) for v in r[:3]) for r in info if r[3]]
            print(f"[bench] rank {rank}: expired waits (site, seen, target): {waits}", file=sys.stderr, flush=True)
            raise RuntimeError(f"rank {rank}: device error flags {ef} after the {phase}")

    for k in range(args.warmup):
        step(k)
    E.emb_join(ex.ctx, stream)
    check_err("warm-up")

    # CUDA graph of G steps = whole cycles of the nb batches (device-resident iteration counter ->
    # replay-safe).  A graph ends with emb_join, which drains the pipeline (the next batch's sort,
    # the last step's deferred part); G >= 64 steps makes that drain one per >= 64 steps, as in a
    # training loop that never joins, instead of one per cycle of nb.
    G = nb * max(1, int(os.environ.get("BENCH_GRAPH_MIN_STEPS", "64")) // nb)
    graph = graph_rem = graph_comp = None
    k0 = args.warmup
    if not args.no_graph:
        try:
            g = torch.cuda.CUDAGraph()
            cap_stream = torch.cuda.Stream()
            cap_stream.wait_stream(stream)
            with torch.cuda.graph(g, stream=cap_stream):
                for j in range(G):
                    b = (k0 + j) % nb
                    if not args.graph_no_prefetch:   # the paper's prefetch, as in step()
                        E.emb_prefetch(ex.ctx, ids_d[(b + 1) % nb], cap_stream)
                    E.emb_forward_exchange(ex.ctx, ids_d[b], Y_d[b], cap_stream)
                    E.emb_backward_exchange(ex.ctx, dY_d[b], ids_d[(b + 1) % nb], cap_stream)
                E.emb_join(ex.ctx, cap_stream)
            stream.wait_stream(cap_stream)
            graph = g
            # K not a multiple of G: the remaining steps (the first K mod G of the graph's sequence) are a
            # graph too (graph_rem), with its complement (the other G - rem steps,
            # graph_comp) so that both can be warmed up before the timed region as one full cycle,
            # and the sequence closed after it (host and device stay one whole cycle apart: same
            # batch, same parity).  Every timed step runs a captured, already-launched graph.
            rem0 = args.steps % G

            def capture(j0, n):
                gg = torch.cuda.CUDAGraph()
                cap_stream.wait_stream(stream)
                with torch.cuda.graph(gg, stream=cap_stream):
                    for j in range(j0, j0 + n):
                        b = (k0 + j) % nb
                        if not args.graph_no_prefetch:
                            E.emb_prefetch(ex.ctx, ids_d[(b + 1) % nb], cap_stream)
                        E.emb_forward_exchange(ex.ctx, ids_d[b], Y_d[b], cap_stream)
                        E.emb_backward_exchange(ex.ctx, dY_d[b], ids_d[(b + 1) % nb], cap_stream)
                    E.emb_join(ex.ctx, cap_stream)
                stream.wait_stream(cap_stream)
                return gg

            if rem0 and os.environ.get("BENCH_GRAPH_REM", "1") != "0":
                graph_rem = capture(0, rem0)
                graph_comp = capture(rem0, G - rem0)
            torch.cuda.synchronize()
            graph.replay()          # one untimed replay (it is also a warm-up cycle)
            if graph_rem is not None:
                graph_rem.replay()  # ... and one of the split cycle
                graph_comp.replay()
            torch.cuda.synchronize()
        except Exception as e:  # pragma: no cover
            print(f"[bench] graph capture failed, timing eagerly: {e}", file=sys.stderr)
            graph = None

    # ---------------- timed region
    K = args.steps
    n_rep, rem = (divmod(K, G) if graph is not None else (0, K))
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st0 = ex.stats() if world > 1 else None
    nv0 = nvlink_kib(local) if world > 1 else None
    clk = ClockSampler(local)  # NVML init here, outside the timed region (it takes milliseconds)
    device_align()
    # ~1 ms of device sleep queued ahead of the start event: the host enqueues the start event and the
    # first replays while the device sleeps, so host launch latency (and the clock sampler's start)
    # never shows up as idle device time inside the timed region; at N > 1 the ranks leave the sleep
    # together (same cycle count after the aligning all_reduce)
    torch.cuda._sleep(2_000_000)
    with clk:
        ev0.record(stream)
        for _ in range(n_rep):
            graph.replay()
        if graph_rem is not None:
            graph_rem.replay()
        else:
            for j in range(rem):
                step(k0 + j)
        E.emb_join(ex.ctx, stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    nv1 = nvlink_kib(local) if world > 1 else None
    barrier()
    ms = ev0.elapsed_time(ev1)
    nvl_meas = None
    if world > 1:
        st1 = ex.stats()
        remote = {k: sum(st1[k][s_] - st0[k][s_] for s_ in range(world) if s_ != rank) / K
                  for k in ("fwd_bytes_pulled", "bwd_bytes_pushed", "ids_bytes_pushed")}
        nvl_meas = {"source": "NVML NVLINK_THROUGHPUT_DATA_TX/RX (all links, KiB counters) around the timed region",
                    "library_counters_per_step": {k: int(v) for k, v in remote.items()},
                    "library_note": "emb_get_stats deltas to/from peers: forward bytes PULLED (arrive as RX), "
                                    "gradient + id bytes PUSHED (leave as TX)"}
        if nv0 and nv1:
            tx, rx = (nv1[0] - nv0[0]) * 1024 / K, (nv1[1] - nv0[1]) * 1024 / K
            nvl_meas.update({"tx_bytes_per_step": int(tx), "rx_bytes_per_step": int(rx),
                             "tx_gbs": round(tx / (ms / K * 1e-3) / 1e9, 1),
                             "rx_gbs": round(rx / (ms / K * 1e-3) / 1e9, 1)})
        else:
            nvl_meas["unavailable"] = "NVML NVLink throughput fields not readable on this host"
    check_err("timed region")
    if os.environ.get("EMB_TRACE_OUT"):  # kernel trace ring (EMB_TRACE builds; scripts/trace.py)
        np.save(f"{os.environ['EMB_TRACE_OUT']}.{rank}.npy", E.emb_debug_copy(ex.ctx, E.EMB_DBG_TIMESTAMPS))
    kk = k0 + rem                  # next batch index (graph replays are whole cycles)
    if graph_rem is not None:      # close the split cycle (untimed)
        graph_comp.replay()
        kk = k0 + G
    t_max = ms
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_max = float(tt.item())
    nonpad = sum(count_nonpad(ids_all[(k0 + j) % nb][s])
                 for j in range(K) for s in range(world))   # cycles are whole, so batch order is irrelevant
    value = nonpad / (t_max / 1e3)

    # ---------------- step-time distribution, with and without the CUDA graph:
    # per-replay events (one cycle of nb steps each) and per-step events of an eager pass; every
    # step's batch index stays in sequence (replays are whole cycles, eager steps continue from kk)
    def _max_over_ranks(xs):
        if world == 1:
            return xs
        tt = torch.tensor(xs, device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        return tt.tolist()

    dist_t = {}
    R = max(4, min(64, K // max(G, 1)))
    if graph is not None:
        # realign the batch sequence with the captured cycle (the graph's first
        # forward expects the ids promised by the step before it)
        for j in range((k0 - kk) % nb):
            step(kk + j)
        kk += (k0 - kk) % nb
        barrier()
        device_align()
        torch.cuda._sleep(2_000_000)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(R + 1)]
        evs[0].record(stream)
        for i in range(R):
            graph.replay()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        per = _max_over_ranks([evs[i].elapsed_time(evs[i + 1]) * 1e3 / G for i in range(R)])
        dist_t["graph"] = {"mean_us": round(statistics.mean(per), 3), "median_us": round(statistics.median(per), 3),
                           "samples": R, "unit": "us per step (per-replay events / steps per replay)"}
    Ee = min(K, 400)
    barrier()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(Ee + 1)]
    evs[0].record(stream)
    for j in range(Ee):
        step(kk + j)
        evs[j + 1].record(stream)
    E.emb_join(ex.ctx, stream)
    e_end = torch.cuda.Event(enable_timing=True)
    e_end.record(stream)
    torch.cuda.synchronize()
    per = _max_over_ranks([evs[j].elapsed_time(evs[j + 1]) * 1e3 for j in range(Ee)])
    tot = _max_over_ranks([evs[0].elapsed_time(e_end) * 1e3 / Ee])[0]
    dist_t["eager"] = {"mean_us": round(tot, 3), "median_us": round(statistics.median(per), 3), "samples": Ee,
                       "unit": "us per step (mean = whole pass incl. deferred tail / steps; median of per-step "
                               "events on the caller's stream)"}
    kk += Ee
    check_err("step-time distribution")

    # ---------------- per-kernel CUDA-event profile (separate, eager, not part of `value`)
    E.emb_profile(ex.ctx, True)
    P = args.profile_steps
    for j in range(P):
        step(kk + j)
    E.emb_join(ex.ctx, stream)
    prof = E.emb_profile_read(ex.ctx)
    E.emb_profile(ex.ctx, False)
    check_err("profile")
    # kernels per step: count the profiled launches (one step = one fwd + one bwd)
    per_step_launch = sum(c for (_, c) in prof.values()) / P
    k_prof = kk
    kk += P

    # ---------------- the same per-kernel events INSIDE a CUDA graph of the timed step: the library
    # records its profiling events as event-record nodes while the stream is captured, so each
    # kernel is timed in the graph structure `value` is measured with (no eager launch path, no host
    # gaps; the event nodes only cut the PDL overlap next to each kernel).  The last of 3 replays
    # is read.  This is the `roofline` timing; the eager pass above stays in `kernels`.
    gprof = None
    if graph is not None:
        for j in range((k0 - kk) % nb):
            step(kk + j)
        kk += (k0 - kk) % nb
        E.emb_join(ex.ctx, stream)
        torch.cuda.synchronize()
        try:
            g2 = torch.cuda.CUDAGraph()
            cap2 = torch.cuda.Stream()
            cap2.wait_stream(stream)
            E.emb_profile(ex.ctx, True)
            with torch.cuda.graph(g2, stream=cap2):
                for j in range(nb):
                    b = (kk + j) % nb
                    E.emb_prefetch(ex.ctx, ids_d[(b + 1) % nb], cap2)
                    E.emb_forward_exchange(ex.ctx, ids_d[b], Y_d[b], cap2)
                    E.emb_backward_exchange(ex.ctx, dY_d[b], ids_d[(b + 1) % nb], cap2)
                E.emb_join(ex.ctx, cap2)
            E.emb_profile(ex.ctx, False)
            stream.wait_stream(cap2)
            for _ in range(3):
                g2.replay()
            torch.cuda.synchronize()
            gprof = E.emb_profile_read(ex.ctx)
            del g2
            check_err("in-graph profile")
        except Exception as e:  # pragma: no cover
            E.emb_profile(ex.ctx, False)
            print(f"[bench] in-graph kernel profile failed: {e}", file=sys.stderr)
            gprof = None

    # algorithmic bytes per kernel, averaged over the profiled batches
    alg = {}
    for j in range(P):
        b = (k_prof + j) % nb
        for kname, (hb, nv) in algorithmic_bytes(cfg, world, rank, ids_all[b], ids_all[(b + 1) % nb],
                                                 mode).items():
            a = alg.setdefault(kname, [0, 0])
            a[0] += hb / P
            a[1] += nv / P
    kern = {}
    for kname, (tot_ms, cnt) in prof.items():
        avg_us = tot_ms / cnt * 1e3
        hb, nv = alg.get(kname, (0, 0))
        kern[kname] = {"avg_us": round(avg_us, 3), "launches": cnt, "hbm_bytes": int(hb), "nvlink_bytes": int(nv),
                       "hbm_gbs": round(hb / (avg_us * 1e-6) / 1e9, 1) if avg_us > 0 else None}
        if gprof and kname in gprof and gprof[kname][1] > 0:
            gus = gprof[kname][0] / gprof[kname][1] * 1e3
            kern[kname]["avg_us_in_graph"] = round(gus, 3)
            kern[kname]["hbm_gbs_in_graph"] = round(hb / (gus * 1e-6) / 1e9, 1) if gus > 0 else None
    timing_note = "eager pass, CUDA events around each launch on its own stream"
    # dominant kernel: the one that must move the most algorithmic bytes
    dom = max(kern, key=lambda k: kern[k]["hbm_bytes"] + kern[k]["nvlink_bytes"])
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    nvl_peak = 770.0  # measured peer copy GB/s per direction (B200_PROFILING.md)
    dk = kern[dom]
    dom_us = dk["avg_us"]
    if dk.get("avg_us_in_graph"):
        dom_us = dk["avg_us_in_graph"]
        timing_note = (f"CUDA events recorded as event-record nodes around each launch inside a CUDA graph of {nb} "
                       "steps (the timed step's structure, last of 3 replays); eager-pass value in kernels.avg_us")
    nvl_gbs = dk["nvlink_bytes"] / (dom_us * 1e-6) / 1e9 if dom_us > 0 else 0
    hbm_gbs = dk["hbm_bytes"] / (dom_us * 1e-6) / 1e9 if dom_us > 0 else 0
    bound = "hbm" if (hbm_gbs / hbm_peak) >= (nvl_gbs / nvl_peak) or world == 1 else "nvlink"
    roof = {"bound": bound, "kernel": dom,
            "achieved": round(hbm_gbs if bound == "hbm" else nvl_gbs, 1),
            "peak": hbm_peak if bound == "hbm" else nvl_peak, "unit": "GB/s",
            "frac": round((hbm_gbs / hbm_peak) if bound == "hbm" else (nvl_gbs / nvl_peak), 4),
            "traffic": traffic_for(args.config, world, dom),
            "avg_us": round(dom_us, 3), "timing": timing_note,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if bound == "hbm" else
            "B200_PROFILING.md measured peer copy 770 GB/s/direction"}

    # whole-step roofline (t_roof / t_measured), SURVEY §8(d)
    step_hbm = sum(v[0] for v in alg.values())
    step_nvl = sum(v[1] for v in alg.values())
    t_roof_us = max(step_hbm / (hbm_peak * 1e9), step_nvl / (nvl_peak * 1e9) if world > 1 else 0) * 1e6
    # forward NVLink bytes, two conventions: the volume a deduplicating pull must
    # move ((N-1) * distinct rows * d * e, counted above) and SURVEY §8(d)'s plain
    # AlltoAll ((N-1) * T_r * d * e, the paper's forward, reading R10)
    esz_ = 2 if cfg.dtype == "bf16" else 4
    fwd_plain = sum((world - 1) * len(ids_all[(k_prof + j) % nb][rank]) * (cfg.D // world) * esz_
                    for j in range(P)) / P
    step_nvl_plain = step_nvl - alg.get("fwd_pull_gather", (0, 0))[1] + fwd_plain
    t_roof_plain_us = max(step_hbm / (hbm_peak * 1e9), step_nvl_plain / (nvl_peak * 1e9) if world > 1 else 0) * 1e6
    ms_per_step = t_max / K

    # ---------------- end to end through the C ABI with host buffers (pinned)
    Ke = min(K, 200)
    h_ids = [x.cpu().pin_memory() for x in ids_d]
    h_dY = [x.cpu().pin_memory() for x in dY_d]
    h_Y = [torch.empty(y.shape, dtype=y.dtype).pin_memory() for y in Y_d]
    h2d = d2h = 0
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # Three-stage pipeline: H2D of step j+1 (copy stream) and D2H of step j
    # (second copy stream) overlap the compute on `stream` and each other
    # (PCIe is full duplex).  Buffer reuse follows embrace.h's borrow rule: a
    # buffer borrowed at step t may be rewritten once `stream` has passed
    # backward(t+1) (event done[t+1]).  ids of step j live in ids_buf[j % 4]
    # (borrowed at j-1 as next_ids and at j as ids), dY in dY_buf[j % 3], Y in
    # Y_buf[j % 3] (read back by the D2H stream).
    NI, NB = 4, 3
    ids_buf = [torch.empty(cfg.max_tokens, dtype=torch.int32, device=dev) for _ in range(NI)]
    dY_buf = [torch.empty((cfg.max_tokens, cfg.D), dtype=tdt, device=dev) for _ in range(NB)]
    Y_buf = [torch.empty((cfg.max_tokens, cfg.D), dtype=tdt, device=dev) for _ in range(NB)]
    s_h2d, s_d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev = lambda: torch.cuda.Event()  # noqa: E731
    in_ready, done, out_done = {}, {}, {}
    device_align()
    e0.record(stream)
    s_h2d.wait_event(e0)
    s_d2h.wait_event(e0)

    def stage_in(j):
        # ids(j+1) (and ids(0) at j = 0) plus dY(j)
        b, bn = (kk + j) % nb, (kk + j + 1) % nb
        nonlocal_h2d = 0
        with torch.cuda.stream(s_h2d):
            if j - 2 in done:
                # dY_buf[j % 3] and ids_buf[(j+1) % 4] were last borrowed at step j-3
                s_h2d.wait_event(done[j - 2])
            if j == 0:
                ids_buf[0][:h_ids[b].numel()].copy_(h_ids[b], non_blocking=True)
                nonlocal_h2d += h_ids[b].numel() * 4
            ids_buf[(j + 1) % NI][:h_ids[bn].numel()].copy_(h_ids[bn], non_blocking=True)
            dY_buf[j % NB][:h_dY[b].shape[0]].copy_(h_dY[b], non_blocking=True)
            nonlocal_h2d += h_ids[bn].numel() * 4 + h_dY[b].numel() * h_dY[b].element_size()
            in_ready[j] = ev()
            in_ready[j].record(s_h2d)
        return nonlocal_h2d

    h2d += stage_in(0)
    for j in range(Ke):
        b, bn = (kk + j) % nb, (kk + j + 1) % nb
        n, nn = h_ids[b].numel(), h_ids[bn].numel()
        cur, nxt = ids_buf[j % NI][:n], ids_buf[(j + 1) % NI][:nn]
        stream.wait_event(in_ready[j])
        if j - NB in out_done:
            stream.wait_event(out_done[j - NB])  # Y_buf[j % 3] read back
        yb = Y_buf[j % NB]
        E.emb_prefetch(ex.ctx, nxt, stream)
        E.emb_forward_exchange(ex.ctx, cur, yb[:n], stream)
        fwd_done = ev()
        fwd_done.record(stream)
        E.emb_backward_exchange(ex.ctx, dY_buf[j % NB][:n], nxt, stream)
        done[j] = ev()
        done[j].record(stream)
        if j + 1 < Ke:
            h2d += stage_in(j + 1)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(fwd_done)
            h_Y[b].copy_(yb[:n], non_blocking=True)
            out_done[j] = ev()
            out_done[j].record(s_d2h)
        d2h += h_Y[b].numel() * h_Y[b].element_size()
    E.emb_join(ex.ctx, stream)
    stream.wait_stream(s_d2h)
    stream.wait_stream(s_h2d)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_tok = sum(count_nonpad(ids_all[(kk + j) % nb][s]) for j in range(Ke) for s in range(world))
    check_err("end-to-end pass")

    # PCIe ceiling of the e2e leg: the same per-step bytes copied with no
    # compute (H2D on s_h2d, D2H on s_d2h, concurrently), pinned host buffers.
    hb_in = torch.empty(max(1, h2d // Ke), dtype=torch.uint8).pin_memory()
    hb_out = torch.empty(max(1, d2h // Ke), dtype=torch.uint8).pin_memory()
    db_in = torch.empty(hb_in.numel(), dtype=torch.uint8, device=dev)
    db_out = torch.empty(hb_out.numel(), dtype=torch.uint8, device=dev)
    Kp = 50
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    s_h2d.wait_event(p0)
    s_d2h.wait_event(p0)
    for _ in range(Kp):
        with torch.cuda.stream(s_h2d):
            db_in.copy_(hb_in, non_blocking=True)
        with torch.cuda.stream(s_d2h):
            hb_out.copy_(db_out, non_blocking=True)
    stream.wait_stream(s_h2d)
    stream.wait_stream(s_d2h)
    p1.record(stream)
    torch.cuda.synchronize()
    pcie_ms = p0.elapsed_time(p1) / Kp
    if world > 1:
        tt = torch.tensor([pcie_ms], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        pcie_ms = float(tt.item())
    pcie_roof = (e2e_tok / Ke) / (pcie_ms / 1e3)
    ex.flush()
    err = ex.stats()["err_flags"]

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(cfg, 1, mode)
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": {"fp32": "f32", "bf16": "bf16"}[cfg.dtype], "data": "synthetic",
            "config": {"workload": (f"{TABLES} stacked tables of " if TABLES > 1 else "")
                                   + f"{cfg.name}: L={cfg.L} D={cfg.D} {cfg.dtype} table, "
                                   + (f"packed <= {cfg.seq_len} tokens" if cfg.packed else
                                      f"{cfg.batch}x{cfg.seq_len} Zipf({cfg.zipf_s}) ids") + " per rank",
                       "mode": mode, "optim": cfg.optim, "parallelism": f"column-shard x{world}",
                       "batches_cycled": nb, "l2": f"rotating {nb} batches (inputs+outputs "
                       f"{nb * 2 * cfg.max_tokens * cfg.D * (2 if cfg.dtype == 'bf16' else 4) / 2**20:.0f} MiB > 126 MiB L2)",
                       "cuda_graph": graph is not None, "graph_steps": G if graph is not None else 0, "tokens_counted": "non-pad (id 0 = pad)"},
            "roofline": roof,
            "step_roofline": {"t_roof_us": round(t_roof_us, 3), "t_step_us": round(ms_per_step * 1e3, 3),
                              "frac": round(t_roof_us / (ms_per_step * 1e3), 4),
                              "hbm_bytes": int(step_hbm), "nvlink_bytes": int(step_nvl),
                              "fwd_nvlink_convention": "distinct rows: (N-1) u_r d e",
                              "plain_alltoall": {"nvlink_bytes": int(step_nvl_plain),
                                                 "t_roof_us": round(t_roof_plain_us, 3),
                                                 "frac": round(t_roof_plain_us / (ms_per_step * 1e3), 4),
                                                 "fwd_nvlink_convention": "SURVEY §8(d): (N-1) T_r d e"}},
            "step_time": dist_t,
            "nvlink_measured": nvl_meas,
            "kernels": kern,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_tok / (e2e_ms / 1e3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(h2d / Ke), "d2h_bytes_per_step": int(d2h / Ke),
                    "steps": Ke, "pcie_bound": {"value": pcie_roof, "frac": (e2e_tok / (e2e_ms / 1e3)) / pcie_roof,
                                                "copy_ms_per_step": pcie_ms,
                                                "what": "same H2D+D2H bytes per step copied concurrently on the "
                                                        "two copy streams with no compute"},
                    "path": "pinned host ids/dY -> H2D (copy stream) -> emb_forward/backward_exchange -> Y D2H (copy stream), pipelined one step"},
            "gpu_launches": int(round(per_step_launch * K)),
            "gpu_launches_per_step": per_step_launch,
            "clocks": clk.summary(),
            "device_errors": err,
        }
        print(json.dumps(line), flush=True)
    ex.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
