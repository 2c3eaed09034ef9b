"""Thin Python binding of libembrace.so (include/embrace.h).

Argument marshalling only: every step of the exchange runs in the library's
CUDA kernels.  Functions keep the C names.  Tensors are torch tensors on the
context's device; streams default to torch's current stream.  If the shared
library is missing the import fails loudly — there is no fallback path.
"""

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libembrace.so")

EMB_MAX_WORLD = 8
EMB_IPC_HANDLE_BYTES = 64
EMB_UNIQUE_ID_BYTES = 128

STATUS = {0: "EMB_OK", 1: "EMB_ERR_INVALID_ARG", 2: "EMB_ERR_SHAPE", 3: "EMB_ERR_ID_RANGE",
          4: "EMB_ERR_CAPACITY", 5: "EMB_ERR_STATE", 6: "EMB_ERR_CUDA", 7: "EMB_ERR_NCCL",
          8: "EMB_ERR_TIMEOUT"}
EMB_FP32, EMB_BF16 = 0, 1
EMB_SGD, EMB_ADAM, EMB_ADAGRAD = 0, 1, 2
OPTIMS = {"sgd": EMB_SGD, "adam": EMB_ADAM, "adagrad": EMB_ADAGRAD}
EMB_BWD_RAW, EMB_BWD_COAL, EMB_BWD_SPLIT = 0, 1, 2
EMB_DBG_GIDS, EMB_DBG_SLOT_IDS, EMB_DBG_COUNTS, EMB_DBG_PERM, EMB_DBG_ISSUE_LOG, EMB_DBG_TIMESTAMPS, \
    EMB_DBG_ERRINFO = range(7)
EMB_STATE_SHARD, EMB_STATE_ADAM_M, EMB_STATE_ADAM_V = range(3)
MODES = {"raw": EMB_BWD_RAW, "coal": EMB_BWD_COAL, "split": EMB_BWD_SPLIT}

EXPORTED = [
    "emb_status_str", "emb_table_base", "emb_workspace_bytes", "emb_create", "emb_ipc_handle", "emb_get_unique_id",
    "emb_shard_init", "emb_sym_base", "emb_shard_init_colocated", "emb_forward_exchange", "emb_prefetch", "emb_backward_exchange", "dense_allreduce_enqueue",
    "dense_queue_flush", "dense_wait", "emb_flush", "emb_join", "emb_profile", "emb_profile_read",
    "emb_get_stats", "emb_debug_copy", "emb_state_ptr", "emb_queue_issue_order", "emb_shard_destroy",
]


class EmbError(RuntimeError):
    def __init__(self, code, where):
        super().__init__(f"{where}: {STATUS.get(code, code)}")
        self.code = code
        self.name = STATUS.get(code, str(code))


class EmbConfig(ctypes.Structure):
    _fields_ = [("vocab", ctypes.c_int64), ("dim", ctypes.c_int32), ("world", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("device", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("max_tokens", ctypes.c_int32), ("mode", ctypes.c_int32), ("optim", ctypes.c_int32),
                ("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("grad_scale", ctypes.c_float), ("pad_id", ctypes.c_int64),
                ("queue_window", ctypes.c_int32), ("timeout_ms", ctypes.c_int32),
                ("num_tables", ctypes.c_int32), ("table_rows", ctypes.c_int64 * 8)]


class EmbStats(ctypes.Structure):
    W = EMB_MAX_WORLD
    _fields_ = [("iter", ctypes.c_int64), ("world", ctypes.c_int32),
                ("n_tokens", ctypes.c_int32 * W), ("u", ctypes.c_int32 * W), ("p", ctypes.c_int32 * W),
                ("q", ctypes.c_int32 * W), ("fwd_bytes_pulled", ctypes.c_int64 * W),
                ("bwd_bytes_pushed", ctypes.c_int64 * W), ("ids_bytes_pushed", ctypes.c_int64 * W),
                ("err_flags", ctypes.c_int32), ("kernel_launches", ctypes.c_int64)]


KERNEL_NAMES = ["fwd_pull_gather", "sort_unique", "mark_next", "coal_push", "merge_update_prior",
                "defpush", "merge_update_sched", "rawpush", "rawcoal", "split_tables", "peer_gate", "coal_apply"]
EMB_NUM_KERNELS = len(KERNEL_NAMES)


_lib_handle = None


def lib():
    """Load libembrace.so (no fallback: raises if it is missing)."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing — run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, u8p = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(ctypes.c_uint8)
        L.emb_status_str.restype = ctypes.c_char_p
        L.emb_status_str.argtypes = [i32]
        sig = {
            "emb_workspace_bytes": [ctypes.POINTER(EmbConfig), ctypes.POINTER(ctypes.c_size_t),
                                    ctypes.POINTER(ctypes.c_size_t)],
            "emb_create": [ctypes.POINTER(EmbConfig), ctypes.POINTER(vp)],
            "emb_table_base": [vp, i32, ctypes.POINTER(i64)],
            "emb_ipc_handle": [vp, u8p],
            "emb_get_unique_id": [u8p],
            "emb_shard_init": [vp, u8p, u8p, vp, vp],
            "emb_sym_base": [vp, ctypes.POINTER(vp)],
            "emb_shard_init_colocated": [vp, ctypes.POINTER(vp), vp, vp],
            "emb_forward_exchange": [vp, vp, i32, vp, vp],
            "emb_backward_exchange": [vp, vp, vp, i32, vp],
            "emb_prefetch": [vp, vp, i32, vp],
            "dense_allreduce_enqueue": [vp, vp, i64, i32, i32, vp, ctypes.POINTER(i64)],
            "dense_queue_flush": [vp],
            "dense_wait": [vp, i64, vp],
            "emb_flush": [vp, vp],
            "emb_join": [vp, vp],
            "emb_profile": [vp, i32],
            "emb_profile_read": [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)],
            "emb_get_stats": [vp, ctypes.POINTER(EmbStats)],
            "emb_debug_copy": [vp, i32, i32, vp, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)],
            "emb_state_ptr": [vp, i32, ctypes.POINTER(vp)],
            "emb_queue_issue_order": [ctypes.POINTER(i32), i32, i32, ctypes.POINTER(i32)],
            "emb_shard_destroy": [vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = i32
        _lib_handle = L
    return _lib_handle


def _ck(code, where):
    if code != 0:
        raise EmbError(code, where)


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _bytes_arg(b):
    if b is None:
        return None
    buf = (ctypes.c_uint8 * len(b)).from_buffer_copy(bytes(b))
    return ctypes.cast(buf, ctypes.POINTER(ctypes.c_uint8))


def make_config(vocab, dim, world=1, rank=0, device=0, dtype="fp32", max_tokens=4096, mode="split",
                optim="sgd", lr=0.1, beta1=0.9, beta2=0.999, eps=1e-8, grad_scale=0.0, pad_id=-1,
                queue_window=1, timeout_ms=10000, table_rows=None):
    tr = list(table_rows or [])
    return EmbConfig(vocab, dim, world, rank, device, EMB_BF16 if dtype == "bf16" else EMB_FP32, max_tokens,
                     MODES[mode] if isinstance(mode, str) else mode, OPTIMS[optim],
                     lr, beta1, beta2, eps, grad_scale, pad_id, queue_window, timeout_ms,
                     len(tr), (ctypes.c_int64 * 8)(*(tr + [0] * (8 - len(tr)))))


# ---------------------------------------------------------------- C names
def emb_status_str(code):
    return lib().emb_status_str(code).decode()


def emb_workspace_bytes(cfg):
    a, b = ctypes.c_size_t(), ctypes.c_size_t()
    _ck(lib().emb_workspace_bytes(ctypes.byref(cfg), ctypes.byref(a), ctypes.byref(b)), "emb_workspace_bytes")
    return a.value, b.value


def emb_table_base(ctx, k):
    b = ctypes.c_int64()
    _ck(lib().emb_table_base(ctx, int(k), ctypes.byref(b)), "emb_table_base")
    return b.value


def emb_create(cfg):
    h = ctypes.c_void_p()
    _ck(lib().emb_create(ctypes.byref(cfg), ctypes.byref(h)), "emb_create")
    return h


def emb_ipc_handle(ctx):
    out = (ctypes.c_uint8 * EMB_IPC_HANDLE_BYTES)()
    _ck(lib().emb_ipc_handle(ctx, out), "emb_ipc_handle")
    return bytes(out)


def emb_get_unique_id():
    out = (ctypes.c_uint8 * EMB_UNIQUE_ID_BYTES)()
    _ck(lib().emb_get_unique_id(out), "emb_get_unique_id")
    return bytes(out)


def emb_shard_init(ctx, peer_handles, nccl_id, shard_init, stream=None):
    _ck(lib().emb_shard_init(ctx, _bytes_arg(peer_handles), _bytes_arg(nccl_id), _ptr(shard_init),
                             _stream(stream)), "emb_shard_init")


def emb_sym_base(ctx):
    p = ctypes.c_void_p()
    _ck(lib().emb_sym_base(ctx, ctypes.byref(p)), "emb_sym_base")
    return p.value


def emb_shard_init_colocated(ctx, peer_bases, shard_init, stream=None):
    arr = (ctypes.c_void_p * len(peer_bases))(*[b or None for b in peer_bases])
    _ck(lib().emb_shard_init_colocated(ctx, arr, _ptr(shard_init), _stream(stream)), "emb_shard_init_colocated")


def emb_forward_exchange(ctx, ids, out, stream=None):
    _ck(lib().emb_forward_exchange(ctx, _ptr(ids), int(ids.numel()), _ptr(out), _stream(stream)),
        "emb_forward_exchange")


def emb_prefetch(ctx, next_ids, stream=None):
    _ck(lib().emb_prefetch(ctx, _ptr(next_ids), int(next_ids.numel()), _stream(stream)), "emb_prefetch")


def emb_backward_exchange(ctx, grad_out, next_ids=None, stream=None):
    n_next = 0 if next_ids is None else int(next_ids.numel())
    _ck(lib().emb_backward_exchange(ctx, _ptr(grad_out), _ptr(next_ids), n_next, _stream(stream)),
        "emb_backward_exchange")


def dense_allreduce_enqueue(ctx, buf, priority, ready_event=None):
    import torch
    dt = EMB_BF16 if buf.dtype == torch.bfloat16 else EMB_FP32
    t = ctypes.c_int64()
    ev = ctypes.c_void_p(ready_event.cuda_event if ready_event is not None else 0)
    _ck(lib().dense_allreduce_enqueue(ctx, _ptr(buf), buf.numel(), dt, int(priority), ev, ctypes.byref(t)),
        "dense_allreduce_enqueue")
    return t.value


def dense_queue_flush(ctx):
    _ck(lib().dense_queue_flush(ctx), "dense_queue_flush")


def dense_wait(ctx, ticket, stream=None):
    _ck(lib().dense_wait(ctx, int(ticket), _stream(stream)), "dense_wait")


def emb_flush(ctx, stream=None):
    _ck(lib().emb_flush(ctx, _stream(stream)), "emb_flush")


def emb_join(ctx, stream=None):
    _ck(lib().emb_join(ctx, _stream(stream)), "emb_join")


def emb_profile(ctx, enable):
    _ck(lib().emb_profile(ctx, 1 if enable else 0), "emb_profile")


def emb_profile_read(ctx):
    """{kernel name: (total ms, launches)} since profiling was enabled."""
    ms = (ctypes.c_double * EMB_NUM_KERNELS)()
    cnt = (ctypes.c_int64 * EMB_NUM_KERNELS)()
    _ck(lib().emb_profile_read(ctx, ms, cnt), "emb_profile_read")
    return {KERNEL_NAMES[k]: (ms[k], cnt[k]) for k in range(EMB_NUM_KERNELS) if cnt[k]}


def emb_get_stats(ctx):
    s = EmbStats()
    _ck(lib().emb_get_stats(ctx, ctypes.byref(s)), "emb_get_stats")
    N = s.world
    return {"iter": s.iter, "world": N, "n_tokens": list(s.n_tokens[:N]), "u": list(s.u[:N]),
            "p": list(s.p[:N]), "q": list(s.q[:N]), "fwd_bytes_pulled": list(s.fwd_bytes_pulled[:N]),
            "bwd_bytes_pushed": list(s.bwd_bytes_pushed[:N]), "ids_bytes_pushed": list(s.ids_bytes_pushed[:N]),
            "err_flags": s.err_flags, "kernel_launches": s.kernel_launches}


def emb_debug_copy(ctx, item, src=0, cap_elems=1 << 22):
    dt = np.int64 if item in (EMB_DBG_ISSUE_LOG, EMB_DBG_TIMESTAMPS) else np.int32
    buf = np.zeros(cap_elems, dtype=dt)
    n = ctypes.c_size_t()
    _ck(lib().emb_debug_copy(ctx, item, src, buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes, ctypes.byref(n)),
        "emb_debug_copy")
    return buf[: n.value].copy()


class _CAI:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def emb_state_ptr(ctx, item, shape=None, dtype=None):
    """Raw device pointer, or (with shape/dtype) a zero-copy torch view."""
    p = ctypes.c_void_p()
    _ck(lib().emb_state_ptr(ctx, item, ctypes.byref(p)), "emb_state_ptr")
    if shape is None:
        return p.value
    import torch
    if dtype == torch.bfloat16:
        return torch.as_tensor(_CAI(p.value, shape, "<i2"), device="cuda").view(torch.bfloat16)
    return torch.as_tensor(_CAI(p.value, shape, "<f4"), device="cuda")


def emb_queue_issue_order(priorities, window):
    n = len(priorities)
    pr = (ctypes.c_int32 * max(n, 1))(*priorities)
    out = (ctypes.c_int32 * max(n, 1))()
    _ck(lib().emb_queue_issue_order(pr, n, int(window), out), "emb_queue_issue_order")
    return list(out[:n])


def emb_shard_destroy(ctx):
    _ck(lib().emb_shard_destroy(ctx), "emb_shard_destroy")
