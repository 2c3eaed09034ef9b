/*
 * embrace.h — C ABI of the B200-native EmbRace sparse-embedding exchange.
 *
 * The method: EmbRace "Sparsity-aware Hybrid Communication" (arXiv 2110.09132,
 * /root/reference/PAPER.md) — an [L, D] embedding table column-partitioned over
 * N GPUs (§4.1.2), a forward AlltoAll of lookup results and a
 * backward AlltoAll of sparse gradients (§4.1.1/§4.1.3,
 * Fig. 3 caption PAPER.md:262), the vertical split of the coalesced sparse
 * gradient into a prior and a scheduled part (Alg. 1), the
 * modified sparse Adam and a priority-ordered AllReduce
 * queue for dense gradients.
 *
 * Conventions (every call):
 *   - Return emb_status; EMB_OK == 0.  No exceptions, no abort.
 *   - Host-side argument checks fail BEFORE anything is enqueued.
 *   - Device-detected errors (id out of range, prefetched-id mismatch, P2P
 *     wait timeout) set a sticky device flag, reported by emb_get_stats and
 *     emb_flush.  CUDA / NCCL errors poison the context: every later call
 *     returns the same code.
 *   - "device" pointers are CUDA device pointers on the context's device;
 *     "host" pointers are ordinary host memory.  cudaStream_t / cudaEvent_t
 *     are passed as opaque handles (emb_stream_t / emb_event_t).
 *   - One context per rank (one process per GPU).  A context is not
 *     thread-safe.
 *   - Call order: emb_create -> emb_ipc_handle -> (exchange handles over the
 *     process group) -> emb_shard_init -> (emb_forward_exchange ->
 *     emb_backward_exchange)* -> emb_flush -> emb_shard_destroy.
 *
 * Ownership: the library owns the partitioned state — the column shard
 * [L, D/N], the Adam moments and the NVLink-visible exchange buffers — in
 * device memory it allocates itself, because peers read the shard and write
 * the receive buffers through CUDA IPC mappings.
 * emb_state_ptr exposes them (for checkpointing and tests).  Everything else
 * (ids, outputs, output gradients, dense buffers, events) is caller-owned and
 * borrowed only for the duration of the stream work the call enqueues.
 */
#ifndef EMBRACE_H
#define EMBRACE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EMB_MAX_WORLD 8
#define EMB_IPC_HANDLE_BYTES 64
#define EMB_UNIQUE_ID_BYTES 128
#define EMB_MAX_TABLES 8

typedef struct CUstream_st* emb_stream_t; /* == cudaStream_t */
typedef struct CUevent_st* emb_event_t;   /* == cudaEvent_t  */

typedef enum {
  EMB_OK = 0,
  EMB_ERR_INVALID_ARG = 1, /* NULL / negative / unknown enum                        */
  EMB_ERR_SHAPE = 2,       /* D % N != 0, (D/N)*e % 16 != 0, N > D, N > 8, D > 1024 */
  EMB_ERR_ID_RANGE = 3,    /* a token id < 0 or >= L (device-detected, sticky)       */
  EMB_ERR_CAPACITY = 4,    /* n > max_tokens, or the per-source sort does not fit     */
  EMB_ERR_STATE = 5,       /* call order; ids of forward(t+1) != next_ids of bwd(t)  */
  EMB_ERR_CUDA = 6,
  EMB_ERR_NCCL = 7,
  EMB_ERR_TIMEOUT = 8      /* a bounded wait on a peer flag expired (sticky)         */
} emb_status;

typedef enum { EMB_FP32 = 0, EMB_BF16 = 1 } emb_dtype; /* table, wire and output dtype */
/* Sparse optimizers (reading R4).  EMB_ADAGRAD (SURVEY
 * §8(f) NEXT-4; "common sparse optimizer such as Adagrad"):
 * PyTorch Adagrad with lr_decay 0 and initial accumulator 0, s += g^2,
 * w -= lr g / (sqrt(s) + eps); its accumulator is EMB_STATE_ADAM_M.        */
typedef enum { EMB_SGD = 0, EMB_ADAM = 1, EMB_ADAGRAD = 2 } emb_optim;
/* Backward modes (reading R2):
 *   RAW   — plain hybrid communication: uncoalesced dY column slices travel,
 *           the owner coalesces;
 *   COAL  — the sender coalesces (Alg. 1 line 2), one exchange;
 *   SPLIT — the sender coalesces and Alg. 1 splits the rows into the prior
 *           part (rows the next batch reads, exchanged + applied on the
 *           caller's stream) and the scheduled part (exchanged + applied on a
 *           low-priority side stream, finished before forward(t+2) or flush). */
typedef enum { EMB_BWD_RAW = 0, EMB_BWD_COAL = 1, EMB_BWD_SPLIT = 2 } emb_bwd_mode;

typedef struct {
  int64_t vocab;        /* L                                                       */
  int32_t dim;          /* D (full embedding width)                                 */
  int32_t world;        /* N, 1..8                                                  */
  int32_t rank;         /* r, 0..N-1                                                */
  int32_t device;       /* CUDA device ordinal of this rank                         */
  emb_dtype dtype;      /* storage / wire / output dtype; math is fp32              */
  int32_t max_tokens;   /* capacity: tokens per rank per iteration, 1..32768         */
  emb_bwd_mode mode;
  emb_optim optim;
  float lr, beta1, beta2, eps;
  float grad_scale;     /* multiplies the summed sparse gradient; 0 => 1/N (R5)    */
  int64_t pad_id;       /* -1: pad is an ordinary id; >= 0: its gradient is dropped */
  int32_t queue_window; /* dense queue window W >= 1 (reading R16)                  */
  int32_t timeout_ms;   /* bound on every peer-flag wait; 0 => 10000                */
  /* Several tables in ONE exchange (PAPER.md:481 the LM's
   * two tables, PAPER.md:319-320 GNMT's encoder and decoder tables): the tables
   * share D and are stacked row-wise into one [vocab, D] row space, table k at
   * rows [base_k, base_k + table_rows[k]) (emb_table_base).  A batch holding
   * lookups of several tables passes GLOBAL row ids (local id + base_k), so one
   * forward / backward call — one sort, one set of exchanges, one update — serves
   * all tables; per-table outputs are row ranges of `out` / `grad_out`.
   * num_tables = 0: one table of `vocab` rows.                               */
  int32_t num_tables;                 /* 0 or 1..EMB_MAX_TABLES; sum(table_rows) == vocab */
  int64_t table_rows[8];              /* EMB_MAX_TABLES                                   */
} emb_config;

typedef struct {
  int64_t iter;                          /* completed backward calls             */
  int32_t world;
  int32_t n_tokens[EMB_MAX_WORLD];       /* T_s of the last iteration            */
  int32_t u[EMB_MAX_WORLD];              /* |unique grad ids| per source         */
  int32_t p[EMB_MAX_WORLD];              /* prior rows per source (Alg. 1 l.4)   */
  int32_t q[EMB_MAX_WORLD];              /* scheduled rows per source (l.5)      */
  /* cumulative bytes this rank moved, per peer (self included for reference;
   * algorithmic counts taken in the kernels that move them):                  */
  int64_t fwd_bytes_pulled[EMB_MAX_WORLD]; /* lookup slices read from peer s's shard */
  int64_t bwd_bytes_pushed[EMB_MAX_WORLD]; /* gradient slices written to owner s     */
  int64_t ids_bytes_pushed[EMB_MAX_WORLD]; /* token ids written to peer s            */
  int32_t err_flags;                     /* sticky device flags: 1 id range, 2 state, 4 timeout */
  int64_t kernel_launches;               /* cumulative kernels this context launched            */
} emb_stats;

/* Kernel kinds for the optional per-kernel CUDA-event profile.              */
typedef enum {
  EMB_K_FWD = 0,      /* a1-a4 forward pull-gather (+ id all-gather push)        */
  EMB_K_SORT = 1,     /* a6 per-source sort / unique (auxiliary stream)           */
  EMB_K_ROUTE = 2,    /* a5 next-id push (prefetch all-gather) + D_next marks     */
  EMB_K_COAL = 3,     /* a7 + a9 + a10 sender coalesce + prior push               */
  EMB_K_MERGE0 = 4,   /* a11 owner merge + update, prior (or whole) part          */
  EMB_K_DEFPUSH = 5,  /* a12 scheduled rows push                                  */
  EMB_K_MERGE1 = 6,   /* a12 owner merge + update, scheduled part                 */
  EMB_K_RAWPUSH = 7,  /* RAW a10 raw slice push                                   */
  EMB_K_RAWCOAL = 8,  /* RAW owner-side coalesce                                  */
  EMB_K_TABLES = 9,   /* a8 Alg. 1 slot tables P_n ++ D_n (off the critical path) */
  EMB_K_GATE = 10,    /* N > 1 peer-flag gate (one warp: publish + wait)           */
  EMB_K_APPLY = 11,   /* a7 combine + a9/a10 push (N > 1) or a11 update (N == 1)   */
  EMB_NUM_KERNELS = 12
} emb_kernel_kind;

/* Debug items for emb_debug_copy (integer parity tests). `src` selects the
 * source rank n where it applies.  All copies are synchronous.              */
typedef enum {
  EMB_DBG_GIDS = 0,     /* int32 [T_src]  gathered ids of source src (iteration of the last bwd) */
  EMB_DBG_SLOT_IDS = 1, /* int32 [u_src]  source src's unique grad ids in slot order:
                           prior part ascending, then scheduled part ascending      */
  EMB_DBG_COUNTS = 2,   /* int32 [4*N]    per source: T, u, p, nchunks               */
  EMB_DBG_PERM = 3,     /* int32 [T_src]  positions of source src sorted by (dropped, id,
                           position); slot k's rows are perm[seg_start[k] .. seg_end[k]) */
  EMB_DBG_ISSUE_LOG = 4, /* int64 [k]     dense-queue tickets in issue order          */
  EMB_DBG_ERRINFO = 6,   /* int32 [8][4]  the first 8 expired peer/flag waits in expiry order: site
                           code, value seen, target, 1 if set (EMB_ERR_TIMEOUT) */
  EMB_DBG_TIMESTAMPS = 5, /* uint64 [16][20][8] kernel trace ring: [t%16][kernel kind][entered,
                             waited, finished, phase stamps] globaltimer ns (EMB_TRACE builds) */
} emb_debug_item;

typedef enum { EMB_STATE_SHARD = 0, EMB_STATE_ADAM_M = 1 /* Adagrad: accumulator */, EMB_STATE_ADAM_V = 2 } emb_state_item;

typedef struct emb_ctx emb_ctx;

const char* emb_status_str(emb_status s);

/* First global row of table k (num_tables > 0): sum of table_rows[0..k).     */
emb_status emb_table_base(emb_ctx* ctx, int32_t k, int64_t* base);

/* Device bytes the context will allocate (symmetric + local), for capacity
 * planning; no allocation happens.                                           */
emb_status emb_workspace_bytes(const emb_config* cfg, size_t* symmetric_bytes, size_t* local_bytes);

/* Validate cfg, select cfg->device, allocate the library-owned state and
 * streams.  No communication.  The shard is not initialised yet.             */
emb_status emb_create(const emb_config* cfg, emb_ctx** out);

/* CUDA IPC handle (EMB_IPC_HANDLE_BYTES) of this rank's NVLink-visible
 * region; the caller all-gathers the N handles over its process group.       */
emb_status emb_ipc_handle(emb_ctx* ctx, uint8_t* handle_out);

/* NCCL unique id (EMB_UNIQUE_ID_BYTES) for the dense-gradient queue; call on
 * rank 0 and broadcast.                                                      */
emb_status emb_get_unique_id(uint8_t* id_out);

/* a0 of SURVEY §8(a): shard init ("partitioned into processes
 * before the training start").
 *   peer_handles : host, N * EMB_IPC_HANDLE_BYTES, rank order (own ignored)
 *   nccl_id      : host, EMB_UNIQUE_ID_BYTES, or NULL (no dense queue)
 *   shard_init   : device [L, D/N] row-major in cfg->dtype — this rank's
 *                  columns W[:, r*D/N:(r+1)*D/N]; copied (caller keeps it)
 * Adam moments are zeroed and the step counter reset.  Collective: all N
 * ranks must call it (it rendezvous on NCCL when nccl_id != NULL).          */
emb_status emb_shard_init(emb_ctx* ctx, const uint8_t* peer_handles, const uint8_t* nccl_id,
                          const void* shard_init, emb_stream_t stream);

/* Co-located ranks (DESIGN.md §6 "Co-located mode"): the N contexts of ONE
 * process share ONE device, so every N > 1 step of the exchange (id push,
 * peer pull, gradient push, owner merge, scheduled part, flag gates) runs on
 * a single GPU with the same kernels and the same flag protocol; peers'
 * regions are plain device pointers instead of CUDA IPC mappings.  For
 * testing the N > 1 paths without N GPUs; no dense queue (NCCL rejects
 * duplicate devices).
 *   emb_sym_base : out, device base of this context's symmetric region
 *   peer_bases   : host, N device pointers in rank order (emb_sym_base of each
 *                  rank; own entry NULL or its own base); each must live on
 *                  cfg->device
 *   shard_init   : as emb_shard_init; borrowed until `stream` completes
 * Unlike emb_shard_init this does NOT synchronise: each rank's boot barrier
 * waits on device for the others, so the caller must issue this for all N
 * contexts before it synchronises any of their streams, and must drive every
 * later collective call of all N ranks before synchronising (each context's
 * work spins, bounded by timeout_ms, on the others' flags).  The N ranks'
 * streams must run concurrently: with 3 library streams per rank plus the
 * caller's, set CUDA_DEVICE_MAX_CONNECTIONS >= 4N before CUDA initialises
 * (streams aliased onto one hardware queue serialise, and a spinning gate
 * then waits until timeout_ms expires: EMB_ERR_TIMEOUT, never a hang).   */
emb_status emb_sym_base(emb_ctx* ctx, void** base);
emb_status emb_shard_init_colocated(emb_ctx* ctx, void* const* peer_bases, const void* shard_init,
                                    emb_stream_t stream);

/* a1-a4 of SURVEY §8(a): forward exchange of iteration t.
 *   ids : device int32 [n]  this rank's token ids (0 <= id < L)
 *   n   : 0 <= n <= max_tokens
 *   out : device [n, D] row-major in cfg->dtype — full embedding rows
 *         out[j, :] = W[ids[j], :] (every column slice pulled from its owner)
 * Enqueued on `stream`; `out` is valid when the stream reaches the end of
 * this call's work.  If the previous backward received next_ids, `ids` must
 * equal them (checked on device -> EMB_ERR_STATE flag).  Collective.        */
emb_status emb_forward_exchange(emb_ctx* ctx, const int32_t* ids, int32_t n, void* out,
                                emb_stream_t stream);

/* a5-a12 of SURVEY §8(a): backward exchange of iteration t (Alg. 1 and
 * PAPER.md:280 "AlltoAll is called again to exchange sparse gradients").
 *   grad_out : device [n, D] in cfg->dtype, gradient of the last forward's
 *              `out` (same n and ids); borrowed until `stream` completes
 *   next_ids : device int32 [n_next], the ids this rank will pass to the next
 *              forward (the paper's prefetch), or NULL on the
 *              last step (D_next = empty: every row is scheduled, reading R8).
 *              Borrowed: it may be read by the library's streams until the
 *              NEXT emb_backward_exchange call; writes to it must be ordered
 *              on `stream` after that call.
 * Every shard row in U = unique(all ranks' ids, pad dropped if pad_id >= 0)
 * receives one optimizer step with g = grad_scale * sum over ranks of its dY
 * rows.  SPLIT: rows in D_next are updated on `stream`; the rest on the side
 * stream, complete before forward(t+2) and at emb_flush.  Collective.       */
/* Optional: the paper's prefetch ("always keep the data of
 * the next iteration in memory") as an explicit point in the stream.  Call it
 * after backward(t-1) and before forward(t) with the ids of iteration t+1
 * (the same device pointer and count later passed to backward(t) as
 * next_ids), once their values are in place in stream order.  The library
 * starts the next batch's prefetch push, sort and D_next tags at this point
 * (overlapping forward(t)) instead of at backward(t).  Calling it or not
 * never changes values.
 *   errors: EMB_ERR_STATE if called between a forward and its backward or
 *           twice; EMB_ERR_CAPACITY if n_next > max_tokens.                  */
emb_status emb_prefetch(emb_ctx* ctx, const int32_t* next_ids, int32_t n_next, emb_stream_t stream);

emb_status emb_backward_exchange(emb_ctx* ctx, const void* grad_out, const int32_t* next_ids,
                                 int32_t n_next, emb_stream_t stream);

/* a13: dense-gradient AllReduce priority queue.
 *   buf      : device [count] (fp32 or bf16), averaged in place over ranks
 *   priority : lower = sooner (dense blocks in FP order; reading R16)
 *   ready    : event the producer recorded after this block's backward, or NULL;
 *              borrowed: it must stay valid and must not be re-recorded until
 *              the request is issued (the comm stream waits on it at issue time)
 *   ticket   : out, id for dense_wait
 * Issue rule (identical on every rank, a pure function of the enqueue
 * sequence): after each enqueue, while >= W requests are pending, issue the
 * smallest (priority, seq).  Requires nccl_id at shard init.
 * Bounded state: completion events are recycled over a ring of 1024 tickets
 * (EMB_ERR_CAPACITY if the ticket 1024 older is still pending), and the issue
 * log (EMB_DBG_ISSUE_LOG) keeps the first 65536 issues.                     */
emb_status dense_allreduce_enqueue(emb_ctx* ctx, void* buf, int64_t count, emb_dtype dtype,
                                   int32_t priority, emb_event_t ready, int64_t* ticket);
/* Issue every pending request in (priority, seq) order.                      */
emb_status dense_queue_flush(emb_ctx* ctx);
/* Make `consumer` wait for the AllReduce of `ticket` (must be issued, and
 * fewer than 1024 tickets old: EMB_ERR_STATE otherwise).                     */
emb_status dense_wait(emb_ctx* ctx, int64_t ticket, emb_stream_t consumer);

/* Make `stream` wait for all outstanding deferred work (scheduled parts) and
 * the dense queue, then synchronise it; returns the sticky device error as a
 * status (EMB_ERR_ID_RANGE / STATE / TIMEOUT) if one was raised.           */
emb_status emb_flush(emb_ctx* ctx, emb_stream_t stream);

/* Make `stream` wait (no host synchronisation) for all outstanding deferred
 * work, so that work enqueued on it afterwards — or an event recorded on it —
 * follows every update of every iteration so far.                           */
emb_status emb_join(emb_ctx* ctx, emb_stream_t stream);

/* Per-kernel CUDA-event timing: when enabled, every kernel launch is
 * bracketed by events on its own stream (while the stream is being captured
 * into a CUDA graph the events become event-record nodes, re-recorded by every
 * replay).  emb_profile_read synchronises, returns the summed milliseconds and
 * launch counts per emb_kernel_kind (arrays of EMB_NUM_KERNELS) — for a
 * captured graph, of its last replay — and clears the record.              */
emb_status emb_profile(emb_ctx* ctx, int32_t enable);
emb_status emb_profile_read(emb_ctx* ctx, double* ms, int64_t* count);

/* Synchronise the device and read the counters of the last iteration.       */
emb_status emb_get_stats(emb_ctx* ctx, emb_stats* out);

/* Synchronous copy of an integer intermediate (see emb_debug_item) into host
 * memory of `cap` bytes; *n receives the element count.                    */
emb_status emb_debug_copy(emb_ctx* ctx, int32_t item, int32_t src, void* host, size_t cap, size_t* n);

/* Device pointer of library-owned state ([L, D/N]; shard in cfg->dtype, Adam
 * moments fp32).  Valid until emb_shard_destroy.                            */
emb_status emb_state_ptr(emb_ctx* ctx, int32_t item, void** ptr);

/* Pure host function of the dense-queue issue rule (reading R16), exposed so
 * the rule can be checked without a GPU: out[i] = seq issued i-th.          */
emb_status emb_queue_issue_order(const int32_t* priorities, int32_t n, int32_t window, int32_t* out);

emb_status emb_shard_destroy(emb_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* EMBRACE_H */
