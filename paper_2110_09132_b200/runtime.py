"""Process-group bootstrap and a small object wrapper over the C ABI.

PyTorch is plumbing here: device memory for caller tensors, the current
stream, and torch.distributed to exchange the CUDA IPC handles / NCCL unique
id between the N processes (one per GPU).  All exchange work happens in
libembrace.so.
"""

import torch

from . import embrace as E


def exchange_bytes(local, world, group=None):
    """All-gather a small bytes payload over the default process group
    (rank order).  world == 1 -> [local]."""
    if world == 1:
        return [bytes(local)]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, bytes(local), group=group)
    return out


def broadcast_bytes(local, world, src=0, group=None):
    if world == 1:
        return bytes(local)
    import torch.distributed as dist
    obj = [bytes(local) if local is not None else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


class EmbraceExchange:
    """One rank's column shard of an [L, D] table plus the exchange.

    shard_init: device tensor [L, D/N] (this rank's columns), fp32 or bf16.
    """

    def __init__(self, vocab, dim, shard_init, *, world=1, rank=0, device=None, dtype="fp32",
                 max_tokens=4096, mode="split", optim="sgd", lr=0.1, beta1=0.9, beta2=0.999, eps=1e-8,
                 grad_scale=0.0, pad_id=-1, queue_window=1, dense_queue=False, timeout_ms=10000, group=None,
                 table_rows=None):
        device = torch.cuda.current_device() if device is None else device
        self.cfg = E.make_config(vocab, dim, world, rank, device, dtype, max_tokens, mode, optim, lr, beta1, beta2,
                                 eps, grad_scale, pad_id, queue_window, timeout_ms, table_rows)
        self.world, self.rank, self.dim, self.vocab = world, rank, dim, vocab
        self.d = dim // world
        self.tdtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.ctx = E.emb_create(self.cfg)
        self._closed = False
        # borrowed device buffers (embrace.h): next_ids / the prefetch argument
        # may be read by the library's streams until the next backward call
        self._borrowed = []
        if shard_init is None:          # co-located ranks: make_colocated() initialises
            return
        handles = exchange_bytes(E.emb_ipc_handle(self.ctx), world, group)
        nccl_id = None
        if dense_queue:
            nccl_id = broadcast_bytes(E.emb_get_unique_id() if rank == 0 else None, world, 0, group)
        E.emb_shard_init(self.ctx, b"".join(handles), nccl_id, shard_init.contiguous())

    # -------------------------------------------------------------- exchange
    def forward(self, ids, out=None, stream=None):
        if out is None:
            out = torch.empty((ids.numel(), self.dim), dtype=self.tdtype, device=ids.device)
        E.emb_forward_exchange(self.ctx, ids, out, stream)
        return out

    def prefetch(self, next_ids, stream=None):
        E.emb_prefetch(self.ctx, next_ids, stream)
        self._borrowed.append(next_ids)

    def backward(self, grad_out, next_ids=None, stream=None):
        E.emb_backward_exchange(self.ctx, grad_out, next_ids, stream)
        # what the previous backward borrowed is released by this call; keep
        # this call's next_ids (and grad_out, read in stream order) alive
        self._borrowed = [next_ids, grad_out]

    def flush(self, stream=None):
        E.emb_flush(self.ctx, stream)

    def stats(self):
        return E.emb_get_stats(self.ctx)

    def debug(self, item, src=0):
        return E.emb_debug_copy(self.ctx, item, src)

    # -------------------------------------------------------------- state views
    def shard(self):
        return E.emb_state_ptr(self.ctx, E.EMB_STATE_SHARD, (self.vocab, self.d), self.tdtype)

    def adam_m(self):
        return E.emb_state_ptr(self.ctx, E.EMB_STATE_ADAM_M, (self.vocab, self.d), torch.float32)

    def adam_v(self):
        return E.emb_state_ptr(self.ctx, E.EMB_STATE_ADAM_V, (self.vocab, self.d), torch.float32)

    # -------------------------------------------------------------- dense queue
    def dense_enqueue(self, buf, priority, ready_event=None):
        return E.dense_allreduce_enqueue(self.ctx, buf, priority, ready_event)

    def dense_flush(self):
        E.dense_queue_flush(self.ctx)

    def dense_wait(self, ticket, stream=None):
        E.dense_wait(self.ctx, ticket, stream)

    def table_base(self, k):
        """First global row of table k (stacked tables, embrace.h num_tables)."""
        return E.emb_table_base(self.ctx, k)

    def sym_base(self):
        return E.emb_sym_base(self.ctx)

    def close(self):
        if not self._closed:
            E.emb_shard_destroy(self.ctx)
            self._closed = True


def make_colocated(vocab, dim, shards, streams, *, device=None, **kw):
    """N ranks of the exchange in ONE process on ONE device (co-located mode,
    embrace.h emb_shard_init_colocated): rank r holds shards[r] ([L, D/N]) and
    runs on streams[r].  Every N > 1 code path (peer pull, gradient push, owner
    merge, scheduled part, flag gates) runs with the same kernels as across
    GPUs.  The caller must drive all N ranks' calls before synchronising any
    stream, and needs CUDA_DEVICE_MAX_CONNECTIONS >= 4N set before CUDA
    initialises.  Returns the N EmbraceExchange objects (rank order)."""
    N = len(shards)
    device = torch.cuda.current_device() if device is None else device
    exs = [EmbraceExchange(vocab, dim, None, world=N, rank=r, device=device, **kw) for r in range(N)]
    bases = [x.sym_base() for x in exs]
    for r, x in enumerate(exs):
        sh = shards[r].contiguous()
        E.emb_shard_init_colocated(x.ctx, bases, sh, streams[r])
        x._borrowed = [sh]              # read by the stream-ordered copy
    return exs
