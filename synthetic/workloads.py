"""Workload configs and seeded generators (no method arithmetic).

Recipe:
  * ids: Zipf(s) over frequency ranks 1..L-1 mapped to id = rank (a
    frequency-sorted vocabulary), drawn by inverse CDF on the normalised k^-s
    table; id 0 is the pad token.
  * padded configs: each sequence's length ~ U[minlen, S]; positions past it
    hold the pad id (trailing pad).
  * packed config (Transformer): sentences of length U[10, 64] appended until
    the next would exceed max_tokens (varying T per rank).
  * W ~ U[-0.05, 0.05) (fp32, or rounded to bf16 for bf16 configs);
    dY ~ U[-1, 1) in the config dtype.
  * Seeds: master 0x21100913; substream per (config, kind, iteration, rank)
    via numpy SeedSequence.
bf16 values are returned as float32 arrays holding bf16-representable values
plus helpers to get the raw uint16 bit patterns.
"""

from dataclasses import dataclass, field

import numpy as np

MASTER_SEED = 0x21100913
PAD_ID = 0


@dataclass(frozen=True)
class Config:
    name: str
    L: int
    D: int
    dtype: str                 # "fp32" | "bf16"
    batch: int                 # sequences per rank (0 for packed)
    seq_len: int               # S (padded configs) or max_tokens (packed)
    min_len: int
    packed: bool = False
    optim: str = "adam"
    lr: float = 1e-3
    zipf_s: float = 1.0
    dense_blocks: int = 0       # a13 dense queue (synthetic)
    dense_block_elems: int = 0

    @property
    def max_tokens(self):
        return self.seq_len if self.packed else self.batch * self.seq_len


CONFIGS = {
    # BASELINE.json configs[0..4]
    "tiny": Config("tiny", 1000, 16, "fp32", 8, 16, 8, optim="sgd", lr=0.1),
    "lstm_lm": Config("lstm_lm", 793_470, 512, "fp32", 128, 35, 18),
    "gnmt": Config("gnmt", 32_320, 1024, "bf16", 128, 26, 13,
                   dense_blocks=16, dense_block_elems=8_400_000),
    "transformer": Config("transformer", 32_768, 1024, "bf16", 0, 4096, 10, packed=True),
    "bert_large": Config("bert_large", 30_522, 1024, "bf16", 32, 512, 128,
                         dense_blocks=24, dense_block_elems=12_600_000),
}


def get_config(name):
    return CONFIGS[name]


def _rng(cfg_name, kind, it, rank):
    key = [MASTER_SEED, sum(ord(c) * 131 ** i for i, c in enumerate(cfg_name)) % (2 ** 31),
           {"ids": 1, "dY": 2, "W": 3, "dense": 4, "misc": 5}[kind], it, rank]
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(key)))


_ZIPF_CDF = {}


def _zipf_cdf(L, s):
    k = (L, s)
    if k not in _ZIPF_CDF:
        w = np.arange(1, L, dtype=np.float64) ** (-s)   # ranks 1..L-1
        c = np.cumsum(w)
        _ZIPF_CDF[k] = c / c[-1]
    return _ZIPF_CDF[k]


def zipf_ids(rng, n, L, s):
    """n ids in [1, L-1] with P(id = k) ∝ k^-s (inverse CDF)."""
    cdf = _zipf_cdf(L, s)
    u = rng.random(n)
    return (np.searchsorted(cdf, u, side="right") + 1).clip(1, L - 1).astype(np.int32)


def gen_ids(cfg, it, rank):
    """Token ids of one rank for iteration ``it`` (int32, flat)."""
    rng = _rng(cfg.name, "ids", it, rank)
    if cfg.packed:
        out = []
        total = 0
        while True:
            ln = int(rng.integers(cfg.min_len, 65))
            if total + ln > cfg.seq_len:
                break
            out.append(zipf_ids(rng, ln, cfg.L, cfg.zipf_s))
            total += ln
        return np.concatenate(out) if out else np.zeros(0, np.int32)
    ids = zipf_ids(rng, cfg.batch * cfg.seq_len, cfg.L, cfg.zipf_s).reshape(cfg.batch, cfg.seq_len)
    lens = rng.integers(cfg.min_len, cfg.seq_len + 1, size=cfg.batch)
    mask = np.arange(cfg.seq_len)[None, :] >= lens[:, None]
    ids[mask] = PAD_ID
    return ids.reshape(-1).astype(np.int32)


def to_bf16_grid(x):
    """float32 -> nearest bf16 (ties to even), as float32 (input preparation)."""
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return (b.astype(np.uint32) << 16).view(np.float32)


def bf16_bits(x):
    """uint16 bit patterns of bf16-representable float32 values."""
    return (np.asarray(x, np.float32).view(np.uint32) >> 16).astype(np.uint16)


def gen_table(cfg, rows=None):
    """W [L, D] (or only ``rows`` of it, same values) ~ U[-0.05, 0.05)."""
    rng = _rng(cfg.name, "W", 0, 0)
    W = (rng.random((cfg.L, cfg.D), dtype=np.float32) * np.float32(0.1) - np.float32(0.05))
    if cfg.dtype == "bf16":
        W = to_bf16_grid(W)
    return W if rows is None else W[rows]


def gen_dY(cfg, it, rank, T):
    rng = _rng(cfg.name, "dY", it, rank)
    dY = rng.random((T, cfg.D), dtype=np.float32) * np.float32(2.0) - np.float32(1.0)
    if cfg.dtype == "bf16":
        dY = to_bf16_grid(dY)
    return dY


def gen_dense(cfg, block, rank, n):
    rng = _rng(cfg.name, "dense", block, rank)
    x = rng.random(n, dtype=np.float32) * np.float32(2.0) - np.float32(1.0)
    return to_bf16_grid(x) if cfg.dtype == "bf16" else x


@dataclass
class Workload:
    cfg: Config
    N: int
    iters: int
    ids: list = field(default_factory=list)    # ids[it][rank] int32
    dY: list = field(default_factory=list)     # dY[it][rank] float32 [T, D]

    def nonpad_tokens(self, it):
        return int(sum((x != PAD_ID).sum() for x in self.ids[it]))


def make_workload(cfg, N, iters, with_dY=True, ranks=None):
    """Pre-generate ``iters`` iterations of (ids, dY) for ranks 0..N-1 (or only
    the listed ``ranks``; others stay None)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    ranks = range(N) if ranks is None else ranks
    wl = Workload(cfg, N, iters)
    for it in range(iters):
        ids_it = [None] * N
        dy_it = [None] * N
        for r in ranks:
            ids_it[r] = gen_ids(cfg, it, r)
            if with_dY:
                dy_it[r] = gen_dY(cfg, it, r, ids_it[r].size)
        wl.ids.append(ids_it)
        wl.dY.append(dy_it)
    return wl
