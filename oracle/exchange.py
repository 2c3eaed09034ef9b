"""Simulated N-worker Sparsity-aware Hybrid Communication iteration
(oracle; test infrastructure only).

What one training iteration of the embedding path computes, written in the
paper's order (§4.1.3 "Hybrid Architecture"; Fig. 3 caption
PAPER.md:262; Alg. 1; Convergence PAPER.md:592-597):

  S0  shard_r = W[:, r-slice]
  S1  gids = concat_r ids_r, offsets                   (Alg. 1 input "gathered
                                                        training data")
  S2  forward: every shard looks up ALL tokens; AlltoAll #1 redistributes the
      lookup results; rank s concatenates the N column slices -> Y_s
                                                       
  S3  D_next = gathered next batch (empty on the last step)
  S4  sender n: COALESCE its sparse gradient (fp64 sum in position order),
      rounded to the wire dtype                        (Alg. 1 line 2)
  S5  P_n = U_n ∩ D_next, D_n = U_n \\ P_n              (Alg. 1 lines 3-5)
  S6  AlltoAll #2: column slices of the (prior, then scheduled) gradients
      travel to their owners
  S7  owner r merges each row's contributions in ascending source rank,
      scales by grad_scale and applies the sparse optimizer, prior part then
      scheduled part, both with step t
  S8  byte counters (self-delivery excluded)           (Table 2)

Backward modes (reading R2):
  "raw"   plain hybrid communication — uncoalesced slices travel, the owner
          coalesces;
  "coal"  the sender coalesces, single exchange;
  "split" the sender coalesces and Alg. 1 splits it into prior / scheduled.
All three give the same values up to association; in bf16 COAL/SPLIT also
round the sender's coalesced rows to bf16 on the wire.

``dense_reference`` is the plain definition (R1-R3) that the exchange reaches:
Y = W[ids], G = dense scatter-add of dY over the global batch, one sparse
optimizer step on the rows of unique(ids).
"""

from dataclasses import dataclass, field

import numpy as np

from . import collectives, optim, partition, sparse
from .bf16 import round_to


@dataclass
class OptimConfig:
    kind: str = "sgd"            # "sgd" | "adam" | "adagrad" (the accumulator rides in m)
    lr: float = 0.1
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    grad_scale: float = None     # default 1/N (reading R5)


@dataclass
class IterResult:
    N: int
    gids: np.ndarray
    offsets: np.ndarray
    T: np.ndarray                              # tokens per rank
    Y: list                                    # Y[s]: [T_s, D] fp64
    U_n: list = field(default_factory=list)    # ascending unique ids per source (grad rows)
    P_n: list = field(default_factory=list)
    D_n: list = field(default_factory=list)
    u: np.ndarray = None
    p: np.ndarray = None
    q: np.ndarray = None
    P: np.ndarray = None                       # owner prior list (ascending)
    Q: np.ndarray = None                       # owner scheduled list (ascending)
    U: np.ndarray = None                       # all updated rows (ascending) = P ∪ Q
    g: np.ndarray = None                       # [|U|, D] merged, scaled fp64 gradient rows
    sigma_g: np.ndarray = None                 # [|U|, D] scale * sum |terms|
    fwd_bytes: np.ndarray = None               # [N, N] bytes r -> s
    bwd_bytes: np.ndarray = None
    ids_bytes: np.ndarray = None
    sigma_W: np.ndarray = None                 # [|U|, D] first-order magnitudes of the
    sigma_m: np.ndarray = None                 # updated W / m / v rows (comparison metric,
    sigma_v: np.ndarray = None                 # SURVEY §8(c))

    def sent(self, which):
        """Per-rank bytes sent, self excluded."""
        M = {"fwd": self.fwd_bytes, "bwd": self.bwd_bytes, "ids": self.ids_bytes}[which]
        return M.sum(axis=1) - np.diag(M)


_ESIZE = {"fp32": 4, "bf16": 2, "fp64": 8}


def _grad_terms(ids, dY, pad_id):
    """The sparse gradient one rank produces: (ids, dY rows), pad positions
    dropped when pad_id >= 0 (reading R6)."""
    ids = np.asarray(ids, dtype=np.int64)
    dY = np.asarray(dY, dtype=np.float64)
    if pad_id is not None and pad_id >= 0:
        keep = ids != pad_id
        return ids[keep], dY[keep]
    return ids, dY


def _quot_sigma(a, num, mu_num, den2, mu_den2, eps):
    """First-order error magnitude of q = a * num / (sqrt(den2) + eps) when num
    and den2 carry errors proportional to the magnitudes mu_num, mu_den2 of the
    terms summed into them (reading B12):
        |dq| <= a mu_num / (sqrt(den2) + eps) + a num mu_den2 / (2 sqrt(den2) (sqrt(den2) + eps)^2).
    The second term is 0 where den2 == 0 (then num == 0 too)."""
    sd = np.sqrt(den2)
    t1 = a * mu_num / (sd + eps)
    with np.errstate(divide="ignore", invalid="ignore"):
        t2 = np.where(sd > 0, a * num * mu_den2 / (2 * sd * (sd + eps) ** 2), 0.0)
    return t1 + t2


def simulate_iteration(shards, ids, dY, next_ids, t, mode="split", dtype="fp32",
                       opt=None, m=None, v=None, pad_id=-1):
    """One iteration on N simulated workers.

    shards : list of N arrays [L, d_r]  (updated in place; values on the ``dtype`` grid)
    ids    : list of N int arrays, ids[r] = rank r's token ids of iteration t
    dY     : list of N arrays [T_r, D] (values on the ``dtype`` grid)
    next_ids : list of N int arrays (iteration t+1) or None (last step, D_next = ∅)
    t      : Adam step value of this iteration (1-based)
    m, v   : Adam moment shards (updated in place, fp32 storage) or None for SGD
    """
    N = len(shards)
    opt = opt or OptimConfig()
    scale = (1.0 / N) if opt.grad_scale is None else opt.grad_scale
    L = shards[0].shape[0]
    widths = [s.shape[1] for s in shards]
    cols = np.cumsum([0] + widths)
    D = int(cols[-1])
    e = _ESIZE[dtype]

    # S1 — gathered ids (AllGather of the training data)
    T = np.array([len(x) for x in ids], dtype=np.int64)
    gathered = collectives.all_gather([np.asarray(x, np.int64) for x in ids])[0]
    gids = np.concatenate(gathered) if N else np.zeros(0, np.int64)
    offsets = np.concatenate([[0], np.cumsum(T)])
    for x in ids:
        x = np.asarray(x)
        if x.size and (x.min() < 0 or x.max() >= L):
            raise IndexError("token id out of vocabulary range")

    # S2 — forward: shard r looks up all ranks' tokens, AlltoAll #1, concat
    fwd_blocks = [[partition.shard_lookup(shards[r], gathered[s]) for s in range(N)] for r in range(N)]
    recv = collectives.all_to_all(fwd_blocks)          # recv[s][r] = shard_r[ids_s]
    Y = [np.concatenate(recv[s], axis=1) if T[s] else np.zeros((0, D)) for s in range(N)]

    # S3 — next set (global, reading R1); empty on the last step (reading R8)
    if next_ids is None:
        next_set = np.zeros(0, np.int64)
    else:
        next_set = np.unique(np.concatenate([np.asarray(x, np.int64) for x in next_ids]))

    res = IterResult(N=N, gids=gids, offsets=offsets, T=T, Y=Y)

    # S4/S5 — per-sender coalesce + Alg. 1 split
    terms = [_grad_terms(ids[n], dY[n], pad_id) for n in range(N)]
    Gc = []
    for n in range(N):
        ti, tv = terms[n]
        uidx, uval, _ = sparse.coalesce(ti, tv)
        _, uabs, _ = sparse.coalesce_abs(ti, tv)
        if mode in ("coal", "split"):
            uval = round_to(uval, dtype)               # coalesced rows go on the wire
        Gc.append((uidx, uval, uabs))
        if mode == "split":
            prior_mask = np.isin(uidx, next_set)
        else:
            prior_mask = np.ones(uidx.size, dtype=bool)  # one part
        res.U_n.append(uidx)
        res.P_n.append(uidx[prior_mask])
        res.D_n.append(uidx[~prior_mask])
    res.u = np.array([x.size for x in res.U_n], np.int64)
    res.p = np.array([x.size for x in res.P_n], np.int64)
    res.q = np.array([x.size for x in res.D_n], np.int64)

    # S6 — AlltoAll #2: sender n sends owner r the r-slice of its gradient
    # rows; SPLIT sends the prior block first, then the scheduled block
    # (two exchanges); RAW/COAL send one block.  Each block is
    # (row ids, values [c, d_r], |terms| [c, d_r]).
    def slice_block(ids_, vals, absv, r):
        c0, c1 = cols[r], cols[r + 1]
        return (ids_, vals[:, c0:c1], absv[:, c0:c1])

    if mode == "raw":
        parts_send = [[[slice_block(terms[n][0], terms[n][1], np.abs(terms[n][1]), r)
                        for r in range(N)] for n in range(N)]]
    else:
        parts_send = []
        for sel in (("P",) if mode == "coal" else ("P", "D")):
            blocks = []
            for n in range(N):
                uidx, uval, uabs = Gc[n]
                keep = np.isin(uidx, res.P_n[n] if sel == "P" else res.D_n[n])
                blocks.append([slice_block(uidx[keep], uval[keep], uabs[keep], r) for r in range(N)])
            parts_send.append(blocks)
    parts_recv = [collectives.all_to_all(b) for b in parts_send]   # [part][owner][source]

    P = np.unique(np.concatenate(res.P_n)) if N else np.zeros(0, np.int64)
    Q = np.unique(np.concatenate(res.D_n)) if N else np.zeros(0, np.int64)
    res.P, res.Q = P, Q
    res.U = np.unique(np.concatenate([P, Q]))
    res.g = np.zeros((res.U.size, D))
    res.sigma_g = np.zeros((res.U.size, D))
    res.sigma_W = np.zeros((res.U.size, D))
    res.sigma_m = np.zeros((res.U.size, D))
    res.sigma_v = np.zeros((res.U.size, D))
    # the rows each received part covers at every owner
    part_rows = [P, Q] if mode == "split" else [np.unique(np.concatenate([P, Q]))]

    # S7 — owner r: merge in ascending source rank, scale, optimizer step t
    for pi, recv_part in enumerate(parts_recv):
        rows = part_rows[pi]
        if rows.size == 0:
            continue
        for r in range(N):
            c0, c1 = cols[r], cols[r + 1]
            acc = np.zeros((rows.size, c1 - c0))
            sab = np.zeros((rows.size, c1 - c0))
            for n in range(N):                              # ascending source rank
                ids_n, val_n, abs_n = recv_part[r][n]
                if mode == "raw":                           # owner coalesces raw slices
                    ids_n, val_n, _ = sparse.coalesce(ids_n, val_n)
                    _, abs_n, _ = sparse.coalesce(recv_part[r][n][0], recv_part[r][n][2])
                pos = np.searchsorted(rows, ids_n)
                acc[pos] += val_n
                sab[pos] += abs_n
            g_r = scale * acc
            sg_r = abs(scale) * sab
            old_W = np.asarray(shards[r][rows], np.float64)
            m_old = np.asarray(m[r][rows], np.float64) if opt.kind in ("adam", "adagrad") else None
            v_old = np.asarray(v[r][rows], np.float64) if opt.kind == "adam" else None
            if opt.kind == "sgd":
                optim.sgd_apply(shards[r], rows, g_r, opt.lr, store=dtype)
            elif opt.kind == "adagrad":
                optim.adagrad_apply(shards[r], m[r], rows, g_r, opt.lr, opt.eps, store=dtype, sstore="fp32")
            else:
                optim.adam_apply(shards[r], m[r], v[r], rows, g_r, t, opt.lr, opt.beta1, opt.beta2,
                                 opt.eps, store=dtype, mstore="fp32")
            new_W = np.asarray(shards[r][rows], np.float64)
            at = np.searchsorted(res.U, rows)
            res.g[at, c0:c1] = g_r
            res.sigma_g[at, c0:c1] = sg_r
            if opt.kind == "sgd":
                res.sigma_W[at, c0:c1] = np.abs(old_W) + opt.lr * sg_r
            elif opt.kind == "adagrad":
                s_new = np.asarray(m[r][rows], np.float64)
                # dW = lr g / (sqrt(s) + eps): first-order error magnitude from g (sigma_g) and from
                # s = s_old + g^2 (reading B12)
                # (|dW| <= lr for any g: the bound is capped at 2 lr where it is ill-conditioned)
                res.sigma_W[at, c0:c1] = (np.abs(old_W) + np.abs(new_W - old_W)
                                          + np.minimum(2 * opt.lr, _quot_sigma(
                                              opt.lr, np.abs(g_r), sg_r, s_new,
                                              np.abs(m_old) + g_r * g_r + 2 * np.abs(g_r) * sg_r, opt.eps)))
                # accumulator s += g^2: first-order magnitude |s| + 2 |g| sigma_g
                res.sigma_m[at, c0:c1] = s_new + 2 * np.abs(g_r) * sg_r
            else:
                m_new = np.asarray(m[r][rows], np.float64)
                v_new = np.asarray(v[r][rows], np.float64)
                a_t = optim.adam_alpha(t, opt.lr, opt.beta1, opt.beta2)
                # dW = alpha m / (sqrt(v) + eps): first-order error magnitude from the magnitudes
                # summed into m and v (not only |dW|: m cancels when g opposes m; reading B12)
                mu_m = (2 - opt.beta1) * np.abs(m_old) + (1 - opt.beta1) * sg_r
                mu_v = (2 - opt.beta2) * np.abs(v_old) + (1 - opt.beta2) * (g_r * g_r + 2 * np.abs(g_r) * sg_r)
                # (|m| / sqrt(v) <= (1-b1) / sqrt((1-b2)(1-b1^2/b2)) for any gradient history, so |dW| is
                # bounded; the first-order term is capped at twice that bound where it is ill-conditioned,
                # e.g. an exactly cancelled g with v = 0)
                step_max = a_t * (1 - opt.beta1) / np.sqrt((1 - opt.beta2) * (1 - opt.beta1 ** 2 / opt.beta2))
                res.sigma_W[at, c0:c1] = (np.abs(old_W) + np.abs(new_W - old_W)
                                          + np.minimum(2 * step_max,
                                                       _quot_sigma(a_t, np.abs(m_new), mu_m, v_new, mu_v, opt.eps)))
                res.sigma_m[at, c0:c1] = np.abs(m_new) + (1 - opt.beta1) * sg_r
                res.sigma_v[at, c0:c1] = v_new + 2 * (1 - opt.beta2) * np.abs(g_r) * sg_r

    # S8 — byte counters: forward (r -> s) = T_s d_r e; backward (n -> r) =
    # c_n d_r e with c_n = T_n (raw), u_n (coal), p_n + q_n (split); ids T_r * 4
    fwd = np.zeros((N, N), np.int64)
    bwd = np.zeros((N, N), np.int64)
    idb = np.zeros((N, N), np.int64)
    for r in range(N):
        for s in range(N):
            fwd[r, s] = T[s] * widths[r] * e
            c = T[r] if mode == "raw" else res.u[r]
            bwd[r, s] = c * widths[s] * e
            idb[r, s] = T[r] * 4
    res.fwd_bytes, res.bwd_bytes, res.ids_bytes = fwd, bwd, idb
    return res


def dense_reference(W, ids, dY, t, dtype="fp32", opt=None, m=None, v=None, pad_id=-1, N=None):
    """Plain definition on the unpartitioned table.

    R1: Y_r = W[ids_r]
    R2: G = sum_r sum_j e_{ids_r[j]} (x) dY_r[j]   (dense L x D scatter-add)
    R3: one optimizer step on rows U = unique(all ids) with g = scale * G[u]
    W, m, v are updated in place.  Returns (Y list, U, G rows of U).
    """
    opt = opt or OptimConfig()
    Nr = len(ids) if N is None else N
    scale = (1.0 / Nr) if opt.grad_scale is None else opt.grad_scale
    Y = [np.asarray(W[np.asarray(x, np.int64)], np.float64) for x in ids]
    L, D = W.shape
    G = np.zeros((L, D))
    touched = np.zeros(L, dtype=bool)
    for r in range(len(ids)):
        ti, tv = _grad_terms(ids[r], dY[r], pad_id)
        for j in range(ti.size):                      # plain loop scatter-add
            G[ti[j]] += tv[j]
            touched[ti[j]] = True
    U = np.flatnonzero(touched)
    g = scale * G[U]
    if opt.kind == "sgd":
        optim.sgd_apply(W, U, g, opt.lr, store=dtype)
    elif opt.kind == "adagrad":
        optim.adagrad_apply(W, m, U, g, opt.lr, opt.eps, store=dtype, sstore="fp32")
    else:
        optim.adam_apply(W, m, v, U, g, t, opt.lr, opt.beta1, opt.beta2, opt.eps,
                         store=dtype, mstore="fp32")
    return Y, U, g
