"""Sparse optimizer steps (oracle; test infrastructure only).

PAPER.md:592-597 (§5 "Convergence"): "each sparse gradient is divided into
two parts and requires parameter updating twice with sparse optimizer.
Because the common sparse optimizer such as Adagrad and SGD is fully
element-wise, [...] updating embedding matrices with multiple gradient parts
or a whole gradient would lead to the same result.  [...] Most parts of Adam
are element-wise except the state parameter step [...] we modify the Adam
optimizer in PyTorch, updating the step state only at applying the scheduled
part of sparse gradient".

Readings (R3/R4): one step value t per iteration used by BOTH parts
and committed at the final part; Adam in PyTorch's SparseAdam form with
lr 1e-3, betas (0.9, 0.999), eps 1e-8; SGD is w -= lr * g.

All functions update rows ``idx`` of the given arrays in place and return
nothing; ``g`` is the (already merged and scaled) fp64 gradient of those rows.
Storage rounding (``store``: "fp32"/"bf16"/"fp64") is applied to the written
parameter rows; Adam moments are stored fp32 (``mstore``) — both are rounding
points the GPU has (reading R11).
"""

import math

import numpy as np

from .bf16 import round_to


def sgd_apply(W, idx, g, lr, store="fp64"):
    """W[u] <- W[u] - lr * g[u]  (north_star: 'the sum of sparse updates equals
    a dense-gradient SGD step')."""
    idx = np.asarray(idx, dtype=np.int64)
    if idx.size == 0:
        return
    W[idx] = round_to(np.asarray(W[idx], np.float64) - lr * np.asarray(g, np.float64), store)


def adam_alpha(t, lr, beta1, beta2):
    """Bias-corrected step size of PyTorch SparseAdam at step t >= 1:
    alpha_t = lr * sqrt(1 - beta2^t) / (1 - beta1^t), in fp64."""
    if t < 1:
        raise ValueError("Adam step must be >= 1")
    return lr * math.sqrt(1.0 - beta2 ** t) / (1.0 - beta1 ** t)


def adam_apply(W, m, v, idx, g, t, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8,
               store="fp64", mstore="fp64"):
    """One SparseAdam update of rows ``idx`` with step value ``t``:
        m <- m + (1 - beta1)(g - m)
        v <- v + (1 - beta2)(g^2 - v)
        W <- W - alpha_t * m / (sqrt(v) + eps)
    Rows not in ``idx`` are untouched (lazy sparse moments)."""
    idx = np.asarray(idx, dtype=np.int64)
    if idx.size == 0:
        return
    g = np.asarray(g, np.float64)
    m_old = np.asarray(m[idx], np.float64)
    v_old = np.asarray(v[idx], np.float64)
    m_new = m_old + (1.0 - beta1) * (g - m_old)
    v_new = v_old + (1.0 - beta2) * (g * g - v_old)
    a = adam_alpha(t, lr, beta1, beta2)
    W_new = np.asarray(W[idx], np.float64) - a * m_new / (np.sqrt(v_new) + eps)
    m[idx] = round_to(m_new, mstore)
    v[idx] = round_to(v_new, mstore)
    W[idx] = round_to(W_new, store)


def adagrad_apply(W, s, idx, g, lr=1e-2, eps=1e-10, store="fp64", sstore="fp64"):
    """One sparse Adagrad update of rows ``idx`` (PAPER.md:594
    "the common sparse optimizer such as Adagrad [...] is fully element-wise";
    PyTorch Adagrad form, lr_decay 0, initial accumulator 0):
        s <- s + g^2
        W <- W - lr * g / (sqrt(s) + eps)
    Element-wise: updating disjoint row parts separately equals one update."""
    idx = np.asarray(idx, dtype=np.int64)
    if idx.size == 0:
        return
    g = np.asarray(g, np.float64)
    s_new = np.asarray(s[idx], np.float64) + g * g
    W_new = np.asarray(W[idx], np.float64) - lr * g / (np.sqrt(s_new) + eps)
    s[idx] = round_to(s_new, sstore)
    W[idx] = round_to(W_new, store)


class PartialAdam:
    """The paper's modified Adam under reading R3: the step value
    of iteration k is t = committed + 1 for every part of that iteration; the
    counter is committed once, when the final (scheduled) part is applied."""

    def __init__(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, store="fp64", mstore="fp64"):
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps
        self.store, self.mstore = store, mstore
        self.step = 0  # committed steps
        self._touched = set()

    def apply_partial(self, W, m, v, idx, g, is_final_part):
        idx = np.asarray(idx, dtype=np.int64)
        rows = set(int(u) for u in idx)
        if rows & self._touched:
            raise ValueError("double update: parts of one iteration must be disjoint")
        self._touched |= rows
        adam_apply(W, m, v, idx, g, self.step + 1, self.lr, self.beta1, self.beta2, self.eps,
                   self.store, self.mstore)
        if is_final_part:
            self.step += 1
            self._touched = set()
