"""In-box comparison baselines, on the same B200s.

Not the product: these are the two data-parallel alternatives the paper
measures EmbRace against, rebuilt here from PyTorch ops + NCCL collectives
(torch.distributed) so that Table 2's ordering can be checked on NVLink 5
instead of the paper's Ethernet / InfiniBand (§4.1.1 Table
2; PAPER.md:466-470 the baselines of the evaluation):

  allgather  Horovod-AllGather-style sparse aggregation: every rank keeps the
             full [L, D] table (replicated), looks up its
             batch locally, and in the backward pass all-gathers every rank's
             sparse gradient (ids + rows, "AllGather" row of
             Table 2); each rank coalesces the N gathered gradients and
             applies the same sparse optimizer step to its replica.
  allreduce  dense-format AllReduce of the embedding gradient (PAPER.md:226,
             Table 2 "AllReduce" row, the Horovod default for a sparse
             gradient): each rank scatters its gradient into a dense [L, D]
             buffer, AllReduces it, and applies the step to every row any
             rank touched.

Both apply the SAME update as the exchange (sum over ranks, grad_scale 1/N,
PyTorch SparseAdam form, readings R3-R5), so the results are comparable to
the oracle (tests/test_gpu_baselines.py).  fp32 math throughout.
"""

import torch
import torch.distributed as dist


class ReplicatedTable:
    """One rank's full replica of an [L, D] table with Adam / SGD state."""

    def __init__(self, W, optim="adam", lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, world=1, kind="allgather"):
        self.W = W.clone()
        self.L, self.D = W.shape
        self.optim, self.lr, self.b1, self.b2, self.eps = optim, lr, beta1, beta2, eps
        self.world, self.kind = world, kind
        self.scale = 1.0 / world
        self.t = 0
        if optim == "adam":
            self.m = torch.zeros(self.L, self.D, dtype=torch.float32, device=W.device)
            self.v = torch.zeros_like(self.m)
        if kind == "allreduce":
            self.G = torch.zeros(self.L, self.D, dtype=torch.float32, device=W.device)
            self.hit = torch.zeros(self.L, dtype=torch.int32, device=W.device)

    def forward(self, ids):
        return self.W[ids.long()]

    def _apply(self, rows, g):
        """One optimizer step on `rows` with the summed gradient rows g (fp32)."""
        g = g * self.scale
        w = self.W[rows].float()
        if self.optim == "sgd":
            w = w - self.lr * g
        else:
            m = self.m[rows] + (1 - self.b1) * (g - self.m[rows])
            v = self.v[rows] + (1 - self.b2) * (g * g - self.v[rows])
            a = self.lr * (1 - self.b2 ** self.t) ** 0.5 / (1 - self.b1 ** self.t)
            w = w - a * m / (v.sqrt() + self.eps)
            self.m[rows] = m
            self.v[rows] = v
        self.W[rows] = w.to(self.W.dtype)

    def backward(self, ids, dY, max_tokens):
        self.t += 1
        ids = ids.long()
        if self.kind == "allgather":
            n = ids.numel()
            ids_p = torch.full((max_tokens,), -1, dtype=torch.long, device=ids.device)
            ids_p[:n] = ids
            dY_p = torch.zeros(max_tokens, self.D, dtype=dY.dtype, device=dY.device)
            dY_p[:n] = dY
            if self.world > 1:
                all_ids = torch.empty(self.world * max_tokens, dtype=torch.long, device=ids.device)
                all_dY = torch.empty(self.world * max_tokens, self.D, dtype=dY.dtype, device=dY.device)
                dist.all_gather_into_tensor(all_ids, ids_p)
                dist.all_gather_into_tensor(all_dY, dY_p)
            else:
                all_ids, all_dY = ids_p, dY_p
            keep = all_ids >= 0
            rows, inv = torch.unique(all_ids[keep], return_inverse=True)
            g = torch.zeros(rows.numel(), self.D, dtype=torch.float32, device=ids.device)
            g.index_add_(0, inv, all_dY[keep].float())
            self._apply(rows, g)
        else:
            self.G.zero_()
            self.hit.zero_()
            self.G.index_add_(0, ids, dY.float())
            self.hit[ids] = 1
            if self.world > 1:
                dist.all_reduce(self.G)
                dist.all_reduce(self.hit)
            rows = torch.nonzero(self.hit, as_tuple=True)[0]
            self._apply(rows, self.G[rows])
