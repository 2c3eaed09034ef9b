// ctx.cu — C-ABI entry points (include/embrace.h): validation, library-owned
// device state, CUDA IPC peer mapping, stream/event orchestration of the
// exchange kernels, stats and debug access.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/embrace.h"
#include "common.cuh"

// Rows per sender reduce chunk (B5): shorter chunks mean more warps in flight
// for the Zipf tail but more partials to combine for the head (the pad id is
// one huge segment); measured best: 8 up to 8192 tokens per rank, 16 above.
#ifndef EMB_C
#define EMB_C 0
#endif
#include "dense_queue.h"
#include "kernels.cuh"

using namespace emb;

namespace {

enum CtxState { ST_CREATED = 0, ST_READY = 1, ST_AFTER_FWD = 2 };

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int bits_for(long long v) {  // bits needed to represent value v (v >= 0)
  int b = 0;
  while ((1ll << b) <= v) ++b;
  return b < 1 ? 1 : b;
}

struct Plan {
  int N, r, d, esz, cpr, cps, C, max_chunks, max_long, idbits, posbits;
  bool key64;
  size_t sort_smem, route_smem;
  SymLayout lay;
  size_t local_bytes;
};

emb_status make_plan(const emb_config* cfg, Plan* pl) {
  if (!cfg) return EMB_ERR_INVALID_ARG;
  if (cfg->world < 1 || cfg->world > EMB_MAX_WORLD) return EMB_ERR_SHAPE;
  if (cfg->rank < 0 || cfg->rank >= cfg->world) return EMB_ERR_INVALID_ARG;
  if (cfg->vocab < 1 || cfg->vocab >= (1ll << 30)) return EMB_ERR_INVALID_ARG;
  if (cfg->dim < 1 || cfg->max_tokens < 1 || cfg->max_tokens > 32768) return EMB_ERR_CAPACITY;
  if (cfg->dtype != EMB_FP32 && cfg->dtype != EMB_BF16) return EMB_ERR_INVALID_ARG;
  if (cfg->mode < EMB_BWD_RAW || cfg->mode > EMB_BWD_SPLIT) return EMB_ERR_INVALID_ARG;
  if (cfg->optim != EMB_SGD && cfg->optim != EMB_ADAM && cfg->optim != EMB_ADAGRAD) return EMB_ERR_INVALID_ARG;
  if (cfg->queue_window < 0) return EMB_ERR_INVALID_ARG;
  if (cfg->num_tables < 0 || cfg->num_tables > EMB_MAX_TABLES) return EMB_ERR_INVALID_ARG;
  if (cfg->num_tables > 0) {
    long long sum = 0;
    for (int k = 0; k < cfg->num_tables; ++k) {
      if (cfg->table_rows[k] < 1) return EMB_ERR_INVALID_ARG;
      sum += cfg->table_rows[k];
    }
    if (sum != cfg->vocab) return EMB_ERR_SHAPE;
  }
  const int N = cfg->world;
  if (N > cfg->dim || cfg->dim % N != 0) return EMB_ERR_SHAPE;
  pl->N = N;
  pl->r = cfg->rank;
  pl->esz = cfg->dtype == EMB_BF16 ? 2 : 4;
  pl->d = cfg->dim / N;
  if ((pl->d * pl->esz) % 16 != 0) return EMB_ERR_SHAPE;
  pl->cpr = cfg->dim * pl->esz / 16;
  pl->cps = pl->d * pl->esz / 16;
  if (pl->cpr > 256 || cfg->dim > 1024) return EMB_ERR_SHAPE;  // rows up to 4 KB; fp32 sums of D <= 1024
  pl->C = EMB_C > 0 ? EMB_C : (cfg->max_tokens <= 8192 ? 8 : 16);
  pl->max_chunks = cfg->max_tokens + cfg->max_tokens / pl->C + 1;
  pl->max_long = cfg->max_tokens / (pl->C + 1) + 1;
  pl->idbits = bits_for(cfg->vocab);  // the value L itself is the invalid-id sentinel
  pl->posbits = bits_for(cfg->max_tokens - 1);
  pl->key64 = pl->idbits + pl->posbits > 32;  // (id or sentinel L) | pos
  pl->sort_smem = sort_smem_bytes(cfg->max_tokens, pl->key64);
  if (pl->sort_smem > 227 * 1024) return EMB_ERR_CAPACITY;

  const size_t L = (size_t)cfg->vocab, T = (size_t)cfg->max_tokens;
  SymLayout& y = pl->lay;
  size_t off = 0;
  y.shard = off; off = align_up(off + L * pl->d * pl->esz, 4096);
  y.gids = off;  off = align_up(off + 2 * N * T * 4, 4096);
  y.ntok = off;  off = align_up(off + 2 * N * 4, 256);
  y.recv = off;  off = align_up(off + 2 * N * T * pl->d * pl->esz, 4096);
  y.flags = off; off = align_up(off + sizeof(Flags), 4096);
  y.total = off;

  size_t loc = 0;
  if (cfg->optim == EMB_ADAM) loc += 2 * L * pl->d * 4;
  if (cfg->optim == EMB_ADAGRAD) loc += L * pl->d * 4;
  if (N > 1) loc += 2 * L * N * 8;                               // slotmap
  loc += 2 * L * 4;                                              // nextmark
  loc += 4 * 2 * N * T * 4 + 2 * 2 * N * (T + 1) * 4;            // perm uid upos slot_id | useg chunk_off
  loc += 2 * N * (size_t)pl->max_chunks * 16 + 2 * N * CNT_W * 4 + 2 * N * (size_t)pl->max_long * 4;
  if (cfg->mode != EMB_BWD_RAW) loc += T * cfg->dim * 4;       // gcoal
  loc += 2 * (size_t)pl->max_chunks * cfg->dim * 4;              // scratch
  if (cfg->mode == EMB_BWD_SPLIT && N > 1) loc += 2 * T * cfg->dim * pl->esz;
  if (cfg->mode == EMB_BWD_RAW) loc += 2 * N * T * pl->d * 4;
  pl->local_bytes = loc;
  return EMB_OK;
}

}  // namespace

struct emb_ctx {
  emb_config cfg;
  Plan pl;
  DevCtx dc;
  LaunchCfg lc;
  int state = ST_CREATED;
  emb_status poisoned = EMB_OK;
  char* sym = nullptr;
  bool peer_open[EMB_MAX_WORLD] = {};
  bool colocated = false;  // emb_shard_init_colocated: peers are contexts of this process on this device
  bool sort_join = true;    // N == 1, prefetched: the forward waits for its sort's event (no GATE_SORTED kernel)
  bool fwd_joined = false;  // the last forward did
  bool fwd_dedup1 = false;  // N == 1 joined forward gathers each distinct row once per chunk (knob)
  bool fwd_dedupn = true;   // N > 1 prefetched forward dedups when its sort is already complete (knob)
  std::vector<void*> allocs;
  cudaStream_t side = nullptr;  // scheduled part (lowest priority)
  cudaStream_t aux = nullptr;   // sort of the next batch; N > 1 also prefetch push + D_next tags + tables
  cudaStream_t aux2 = nullptr;  // N == 1: the sorts of odd batches (two sorts may overlap; 8 SMs each);
                                // N > 1 (EMB_SORT_STREAM, one GPU per process): every prefetched sort
  cudaEvent_t ev_gsort = nullptr;  // N > 1: ids of the next batch gathered (aux) -> its sort (aux2)
  cudaEvent_t ev_prior[2] = {}, ev_def[2] = {}, ev_main[2] = {}, ev_sorted[2] = {}, ev_tables[2] = {}, ev_plan[2] = {};
  bool def_pending[2] = {false, false};
  bool sort_pending[2] = {false, false};
  bool tables_pending[2] = {false, false};  // N == 1: tables(t) on the side stream still reads parity t&1
  cudaEvent_t ev_marked = nullptr, ev_join_aux = nullptr, ev_join_side = nullptr, ev_join_aux2 = nullptr;
  bool mark_pending = false;  // N == 1: mark runs on the side stream; the next forward checks its pushed ids
  bool aux_used = false, side_used = false;  // since the last emb_join
  bool aux2_used = false;  // N == 1: a sort went to aux2 since the last emb_join (a capture that never
                           // forked aux2 must not join it: that would depend on uncaptured work)
  long long it = 0;          // forward calls so far (host mirror of the device t)
  long long bwd_done = 0;
  bool prefetched = false;   // last backward pushed next ids
  // emb_prefetch: fork point of the next batch's work, recorded before forward(t)
  const int32_t* pf_ids = nullptr;
  int32_t pf_n = -1;
  bool pf_armed = false;
  cudaEvent_t ev_pre = nullptr;
  bool fwd_pushed = false;   // last forward pushed its ids (route publishes them)
  int last_n = 0;
  DenseQueue* dq = nullptr;
  long long launches = 0;
  bool prof = false;
  struct ProfRec { int kind; cudaEvent_t a, b; };
  std::vector<ProfRec> prof_recs;
};

// Launch one kernel through `fn`, counting it and (when profiling) bracketing
// it with CUDA events on its own stream.
// While the stream is being captured into a CUDA graph the events become
// event-record NODES (cudaEventRecordExternal): every replay re-records them,
// so the kernel is timed inside the graph it is benchmarked in (no host gaps,
// no eager launch path; the event nodes only cut the PDL overlap around it).
static void prof_record(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
  else cudaEventRecord(ev, s);
}

template <typename F>
static cudaError_t run_k(emb_ctx* ctx, int kind, cudaStream_t s, F&& fn) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (ctx->prof) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    prof_record(a, s);
  }
  cudaError_t e = fn();
  ctx->launches += 1;
  if (ctx->prof) {
    prof_record(b, s);
    ctx->prof_recs.push_back({kind, a, b});
  }
  return e;
}

// N > 1 peer-flag gate before a consumer kernel (k_gate.cu); nothing at N == 1
static cudaError_t gate(emb_ctx* ctx, int p, int kind, int flag_arg, cudaStream_t s) {
  if (ctx->pl.N == 1) return cudaSuccess;
  return run_k(ctx, EMB_K_GATE, s, [&] { return launch_gate(ctx->dc, p, kind, flag_arg, s); });
}

#define CKC(ctx, call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      fprintf(stderr, "[embrace] CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      if (ctx) (ctx)->poisoned = EMB_ERR_CUDA;                                          \
      return EMB_ERR_CUDA;                                                              \
    }                                                                                   \
  } while (0)

static int env_int(const char* name, int dflt, int lo, int hi) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  const int x = atoi(v);
  return x < lo ? lo : (x > hi ? hi : x);
}

static emb_status ctx_check(emb_ctx* ctx) {
  if (!ctx) return EMB_ERR_INVALID_ARG;
  if (ctx->poisoned != EMB_OK) return ctx->poisoned;
  return EMB_OK;
}

static cudaError_t dev_alloc(emb_ctx* ctx, void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaSuccess) {
    ctx->allocs.push_back(*p);
    e = cudaMemset(*p, 0, bytes);
  }
  return e;
}

extern "C" {

const char* emb_status_str(emb_status s) {
  switch (s) {
    case EMB_OK: return "EMB_OK";
    case EMB_ERR_INVALID_ARG: return "EMB_ERR_INVALID_ARG";
    case EMB_ERR_SHAPE: return "EMB_ERR_SHAPE";
    case EMB_ERR_ID_RANGE: return "EMB_ERR_ID_RANGE";
    case EMB_ERR_CAPACITY: return "EMB_ERR_CAPACITY";
    case EMB_ERR_STATE: return "EMB_ERR_STATE";
    case EMB_ERR_CUDA: return "EMB_ERR_CUDA";
    case EMB_ERR_NCCL: return "EMB_ERR_NCCL";
    case EMB_ERR_TIMEOUT: return "EMB_ERR_TIMEOUT";
  }
  return "EMB_ERR_UNKNOWN";
}

emb_status emb_table_base(emb_ctx* ctx, int32_t k, int64_t* base) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  const int nt = ctx->cfg.num_tables > 0 ? ctx->cfg.num_tables : 1;
  if (!base || k < 0 || k >= nt) return EMB_ERR_INVALID_ARG;
  long long b = 0;
  for (int i = 0; i < k; ++i) b += ctx->cfg.table_rows[i];
  *base = b;
  return EMB_OK;
}

emb_status emb_workspace_bytes(const emb_config* cfg, size_t* symmetric_bytes, size_t* local_bytes) {
  Plan pl;
  emb_status st = make_plan(cfg, &pl);
  if (st != EMB_OK) return st;
  if (symmetric_bytes) *symmetric_bytes = pl.lay.total;
  if (local_bytes) *local_bytes = pl.local_bytes;
  return EMB_OK;
}

emb_status emb_create(const emb_config* cfg, emb_ctx** out) {
  if (!out) return EMB_ERR_INVALID_ARG;
  *out = nullptr;
  Plan pl;
  emb_status st = make_plan(cfg, &pl);
  if (st != EMB_OK) return st;
  emb_ctx* ctx = new (std::nothrow) emb_ctx();
  if (!ctx) return EMB_ERR_CUDA;
  ctx->cfg = *cfg;
  if (ctx->cfg.queue_window < 1) ctx->cfg.queue_window = 1;
  ctx->pl = pl;
  cudaError_t e = cudaSetDevice(cfg->device);
  if (e != cudaSuccess) { delete ctx; return EMB_ERR_CUDA; }
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cfg->device);
  ctx->lc.nsm = nsm > 0 ? nsm : 148;
  // tuning knobs (measured defaults): forward grid cap per SM,
  // and how a prefetched N == 1 forward orders itself after its sort
  ctx->lc.fwd_per_sm = env_int("EMB_FWD_GRID_PER_SM", 4, 1, 32);
  ctx->lc.reduce_per_sm = env_int("EMB_REDUCE_GRID_PER_SM", 12, 1, 32);
  // N == 1 forward via the bulk-copy engine for tables larger than L2 (rows come
  // from HBM: LM 19.4 vs 19.8 us); for the 32K-row tables, which live in L2,
  // the register gather measured faster (GNMT 19.1 vs 19.6, BERT 44.6 vs 46.4 us;
  // profiles/r02_tune/fwd_bulk.txt).  EMB_FWD_BULK=0/1 overrides.
  {
    const bool big = (double)cfg->vocab * cfg->dim * pl.esz > 96.0 * (1 << 20);
    ctx->lc.fwd_bulk = env_int("EMB_FWD_BULK", big ? 1 : 0, 0, 1);
  }
  ctx->sort_join = env_int("EMB_SORT_JOIN", 1, 0, 1) != 0;
  ctx->fwd_dedup1 = env_int("EMB_FWD_DEDUP1", 0, 0, 1) != 0;
  // N > 1 forward dedup (measured: BERT N = 2 74.3 vs 80.4 us without; LM, GNMT within 1 us)
  ctx->fwd_dedupn = env_int("EMB_FWD_DEDUPN", 1, 0, 1) != 0;  // measured slower at N == 1 (profiles/r02_tune/next3.txt)

  DevCtx& c = ctx->dc;
  memset(&c, 0, sizeof(c));
  c.N = pl.N; c.r = pl.r; c.L = cfg->vocab; c.D = cfg->dim; c.d = pl.d; c.esz = pl.esz;
  c.dtype = cfg->dtype == EMB_BF16 ? BF16 : F32;
  c.mode = (int)cfg->mode; c.optim = cfg->optim == EMB_ADAM ? ADAM : (cfg->optim == EMB_ADAGRAD ? ADAGRAD : SGD);
  c.max_tok = cfg->max_tokens; c.cpr = pl.cpr; c.cps = pl.cps; c.pad_id = cfg->pad_id;
  c.lr = cfg->lr; c.beta1 = cfg->beta1; c.beta2 = cfg->beta2; c.eps = cfg->eps;
  c.scale = cfg->grad_scale != 0.f ? cfg->grad_scale : 1.0f / (float)pl.N;
  c.timeout_ns = (unsigned long long)(cfg->timeout_ms > 0 ? cfg->timeout_ms : 10000) * 1000000ull;
  c.pdl_early = env_int("EMB_PDL_EARLY", 0, 0, 1);
  c.bypass = env_int("EMB_SINGLE_BYPASS", 1, 0, 1);
  c.C = pl.C; c.max_chunks = pl.max_chunks; c.max_long = pl.max_long; c.idbits = pl.idbits; c.posbits = pl.posbits;
  c.lay = pl.lay;

#define ALLOC(ptr, bytes) \
  do { void* p_ = nullptr; if (dev_alloc(ctx, &p_, (bytes)) != cudaSuccess) goto fail; ptr = reinterpret_cast<decltype(ptr)>(p_); } while (0)
  {
    const size_t L = (size_t)cfg->vocab, T = (size_t)cfg->max_tokens, N = pl.N;
    // symmetric region: plain cudaMalloc so it can be IPC-exported
    if (cudaMalloc(reinterpret_cast<void**>(&ctx->sym), pl.lay.total) != cudaSuccess) goto fail;
    // zero ids/ntok/flags now: peers may write into them as soon as handles are exchanged
    if (cudaMemset(ctx->sym + pl.lay.gids, 0, pl.lay.recv - pl.lay.gids) != cudaSuccess) goto fail;
    if (cudaMemset(ctx->sym + pl.lay.flags, 0, sizeof(Flags)) != cudaSuccess) goto fail;
    c.sym[pl.r] = ctx->sym;
    if (cfg->optim == EMB_ADAM) {
      ALLOC(c.adam_m, L * pl.d * 4);
      ALLOC(c.adam_v, L * pl.d * 4);
    }
    if (cfg->optim == EMB_ADAGRAD) ALLOC(c.adam_m, L * pl.d * 4);  // the accumulator
    if (N > 1) ALLOC(c.slotmap, 2 * L * N * 8);
    ALLOC(c.nextmark, 2 * L * 4);
    ALLOC(c.perm, 2 * N * T * 4);
    ALLOC(c.uid, 2 * N * T * 4);
    ALLOC(c.upos, 2 * N * T * 4);
    ALLOC(c.useg, 2 * N * (T + 1) * 4);
    ALLOC(c.slot_id, 2 * N * T * 4);
    if (N > 1) ALLOC(c.plan, 2 * 2 * N * T * (1 + N) * 4);
    ALLOC(c.plan_cnt, 2 * 2 * 4);
    ALLOC(c.chunk_off, 2 * N * (T + 1) * 4);
    ALLOC(c.chunk_desc, 2 * N * (size_t)pl.max_chunks * 16);
    if (cfg->mode != EMB_BWD_RAW) ALLOC(c.gcoal, T * cfg->dim * 4);
    ALLOC(c.long_u, 2 * N * (size_t)pl.max_long * 4);
    ALLOC(c.counts, 2 * N * CNT_W * 4);
    ALLOC(c.scratch, 2 * (size_t)pl.max_chunks * cfg->dim * 4);
    if (cfg->mode == EMB_BWD_SPLIT && N > 1) ALLOC(c.stage, 2 * T * cfg->dim * pl.esz);
    if (cfg->mode == EMB_BWD_RAW) ALLOC(c.gc_owner, 2 * N * T * pl.d * 4);
    ALLOC(c.t_rec, 2 * 4);
    ALLOC(c.sorted, 2 * 4);
    ALLOC(c.sort_cnt, 2 * 4);
    ALLOC(c.sort_count, 2 * 4);
    ALLOC(c.side_it, 4);
    ALLOC(c.marked, 2 * 4);
    ALLOC(c.mark_cnt, 2 * 4);
    ALLOC(c.seq, 4 * 4);
    ALLOC(c.fwd_dd, 2 * 4);
    ALLOC(c.merge_cnt, 2 * 4);
    ALLOC(c.fp, 2 * 4 * 4);
    ALLOC(c.alpha, 2 * 4);
    ALLOC(c.err, 4);
    ALLOC(c.err_info, 33 * 4);
    ALLOC(c.stats, 3 * N * 8);
    ALLOC(c.dbg_ts, EMB_TRACE_SLOTS * 8);
  }
#undef ALLOC
  if (sort_set_smem(cfg->max_tokens, pl.key64, pl.sort_smem) != cudaSuccess) goto fail;
  if (fwd_bulk_set_smem(ctx->dc) != cudaSuccess) goto fail;
  // load every kernel now (see kernels.cuh: preload)
  if (preload_fwd() != cudaSuccess || preload_bwd() != cudaSuccess || preload_route() != cudaSuccess ||
      preload_sort() != cudaSuccess || preload_gate() != cudaSuccess)
    goto fail;
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);  // lo = least priority
    if (cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, lo) != cudaSuccess) goto fail;
    if (cudaStreamCreateWithPriority(&ctx->aux, cudaStreamNonBlocking, hi) != cudaSuccess) goto fail;
    // N == 1 only: at N > 1 every sort runs on aux (co-located ranks keep <= 3 streams each)
    if (pl.N == 1 && cudaStreamCreateWithPriority(&ctx->aux2, cudaStreamNonBlocking, hi) != cudaSuccess) goto fail;
  }
  for (int i = 0; i < 2; ++i) {
    if (cudaEventCreateWithFlags(&ctx->ev_prior[i], cudaEventDisableTiming) != cudaSuccess) goto fail;
    if (cudaEventCreateWithFlags(&ctx->ev_def[i], cudaEventDisableTiming) != cudaSuccess) goto fail;
    if (cudaEventCreateWithFlags(&ctx->ev_main[i], cudaEventDisableTiming) != cudaSuccess) goto fail;
    if (cudaEventCreateWithFlags(&ctx->ev_sorted[i], cudaEventDisableTiming) != cudaSuccess) goto fail;
    if (cudaEventCreateWithFlags(&ctx->ev_tables[i], cudaEventDisableTiming) != cudaSuccess) goto fail;
    if (cudaEventCreateWithFlags(&ctx->ev_plan[i], cudaEventDisableTiming) != cudaSuccess) goto fail;
  }
  if (cudaEventCreateWithFlags(&ctx->ev_marked, cudaEventDisableTiming) != cudaSuccess) goto fail;
  if (cudaEventCreateWithFlags(&ctx->ev_pre, cudaEventDisableTiming) != cudaSuccess) goto fail;
  if (cudaEventCreateWithFlags(&ctx->ev_join_aux, cudaEventDisableTiming) != cudaSuccess) goto fail;
  if (cudaEventCreateWithFlags(&ctx->ev_join_aux2, cudaEventDisableTiming) != cudaSuccess) goto fail;
  if (cudaEventCreateWithFlags(&ctx->ev_gsort, cudaEventDisableTiming) != cudaSuccess) goto fail;
  if (cudaEventCreateWithFlags(&ctx->ev_join_side, cudaEventDisableTiming) != cudaSuccess) goto fail;
  if (cudaDeviceSynchronize() != cudaSuccess) goto fail;
  *out = ctx;
  return EMB_OK;
fail:
  fprintf(stderr, "[embrace] emb_create failed: %s\n", cudaGetErrorString(cudaGetLastError()));
  for (void* p : ctx->allocs) cudaFree(p);
  if (ctx->sym) cudaFree(ctx->sym);
  delete ctx;
  return EMB_ERR_CUDA;
}

emb_status emb_ipc_handle(emb_ctx* ctx, uint8_t* handle_out) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (!handle_out) return EMB_ERR_INVALID_ARG;
  static_assert(sizeof(cudaIpcMemHandle_t) == EMB_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  CKC(ctx, cudaSetDevice(ctx->cfg.device));
  CKC(ctx, cudaIpcGetMemHandle(&h, ctx->sym));
  memcpy(handle_out, &h, sizeof(h));
  return EMB_OK;
}

emb_status emb_get_unique_id(uint8_t* id_out) {
  if (!id_out) return EMB_ERR_INVALID_ARG;
  static_assert(sizeof(ncclUniqueId) == EMB_UNIQUE_ID_BYTES, "nccl id size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return EMB_ERR_NCCL;
  memcpy(id_out, &id, sizeof(id));
  return EMB_OK;
}

// boot barrier over the flags region: every rank stores 1 into every peer's
// boot slot after its shard copy, then waits for all (bounded).
__global__ void boot_kernel(DevCtx c, uint32_t val) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int s = 0; s < c.N; ++s) st_release_sys(&flags_of(c, s)->boot[c.r], val);
  for (int s = 0; s < c.N; ++s) wait_flag(c, &flags_of(c, c.r)->boot[s], val, 12 * 16 + s);
}

// shard copy, zeroed moments and the boot barrier (every rank's shard loaded)
static emb_status shard_load(emb_ctx* ctx, const void* shard_init, cudaStream_t stream) {
  const size_t shard_bytes = (size_t)ctx->cfg.vocab * ctx->pl.d * ctx->pl.esz;
  CKC(ctx, cudaMemcpyAsync(ctx->sym + ctx->pl.lay.shard, shard_init, shard_bytes, cudaMemcpyDeviceToDevice, stream));
  if (ctx->dc.adam_m) CKC(ctx, cudaMemsetAsync(ctx->dc.adam_m, 0, (size_t)ctx->cfg.vocab * ctx->pl.d * 4, stream));
  if (ctx->dc.adam_v) CKC(ctx, cudaMemsetAsync(ctx->dc.adam_v, 0, (size_t)ctx->cfg.vocab * ctx->pl.d * 4, stream));
  boot_kernel<<<1, 32, 0, stream>>>(ctx->dc, 1u);
  CKC(ctx, cudaGetLastError());
  return EMB_OK;
}

emb_status emb_sym_base(emb_ctx* ctx, void** base) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (!base) return EMB_ERR_INVALID_ARG;
  *base = ctx->sym;
  return EMB_OK;
}

emb_status emb_shard_init_colocated(emb_ctx* ctx, void* const* peer_bases, const void* shard_init,
                                    emb_stream_t stream_) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (ctx->state != ST_CREATED) return EMB_ERR_STATE;
  if (!shard_init || !peer_bases) return EMB_ERR_INVALID_ARG;
  CKC(ctx, cudaSetDevice(ctx->cfg.device));
  for (int s = 0; s < ctx->pl.N; ++s) {
    if (s == ctx->pl.r) {
      if (peer_bases[s] != nullptr && peer_bases[s] != ctx->sym) return EMB_ERR_INVALID_ARG;
      continue;
    }
    if (!peer_bases[s]) return EMB_ERR_INVALID_ARG;
    cudaPointerAttributes a;
    CKC(ctx, cudaPointerGetAttributes(&a, peer_bases[s]));
    if (a.type != cudaMemoryTypeDevice || a.device != ctx->cfg.device) return EMB_ERR_INVALID_ARG;
    ctx->dc.sym[s] = static_cast<char*>(peer_bases[s]);
  }
  // no host synchronisation: the boot barrier waits on device for the other
  // co-located ranks, whose init the caller issues next (embrace.h)
  st = shard_load(ctx, shard_init, reinterpret_cast<cudaStream_t>(stream_));
  if (st != EMB_OK) return st;
  ctx->colocated = true;
  ctx->state = ST_READY;
  return EMB_OK;
}

emb_status emb_shard_init(emb_ctx* ctx, const uint8_t* peer_handles, const uint8_t* nccl_id,
                          const void* shard_init, emb_stream_t stream_) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (ctx->state != ST_CREATED) return EMB_ERR_STATE;
  if (!shard_init || (ctx->pl.N > 1 && !peer_handles)) return EMB_ERR_INVALID_ARG;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  CKC(ctx, cudaSetDevice(ctx->cfg.device));
  for (int s = 0; s < ctx->pl.N; ++s) {
    if (s == ctx->pl.r) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, peer_handles + (size_t)s * EMB_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    CKC(ctx, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    ctx->dc.sym[s] = static_cast<char*>(p);
    ctx->peer_open[s] = true;
  }
  st = shard_load(ctx, shard_init, stream);
  if (st != EMB_OK) return st;
  CKC(ctx, cudaStreamSynchronize(stream));
  int err = 0;
  CKC(ctx, cudaMemcpy(&err, ctx->dc.err, 4, cudaMemcpyDeviceToHost));
  if (err & ERR_TIMEOUT) { ctx->poisoned = EMB_ERR_TIMEOUT; return EMB_ERR_TIMEOUT; }
  // N > 1, one GPU per process: the prefetched sort of the next batch on a
  // stream of its own (EMB_SORT_STREAM), forked from aux right after the ids
  // gate, so the aux chain (tags, merge plan) no longer waits behind it.  Pays
  // where that chain bounds the step, at N >= 4 (steady state, N = 4: LM 52.7
  // -> 46.9 us, BERT 91 -> 73 us, GNMT / Transformer neutral); mixed at N = 2,
  // so off there — profiles/r02_tune/sort_stream.txt.
  // Not for co-located ranks, which keep <= 3 streams each.
  if (ctx->pl.N > 1 && env_int("EMB_SORT_STREAM", ctx->pl.N >= 4 ? 1 : 0, 0, 1)) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    CKC(ctx, cudaStreamCreateWithPriority(&ctx->aux2, cudaStreamNonBlocking, hi));
  }
  if (nccl_id) {
    ctx->dq = dense_queue_create(nccl_id, ctx->pl.N, ctx->pl.r, ctx->cfg.queue_window);
    if (!ctx->dq) { ctx->poisoned = EMB_ERR_NCCL; return EMB_ERR_NCCL; }
  }
  ctx->state = ST_READY;
  return EMB_OK;
}

emb_status emb_forward_exchange(emb_ctx* ctx, const int32_t* ids, int32_t n, void* out, emb_stream_t stream_) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (ctx->state == ST_CREATED) return EMB_ERR_STATE;
  if (n < 0 || n > ctx->cfg.max_tokens) return EMB_ERR_CAPACITY;
  if (n > 0 && (!ids || !out)) return EMB_ERR_INVALID_ARG;
  if (ctx->state == ST_AFTER_FWD) return EMB_ERR_STATE;  // backward of the previous forward missing
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  ctx->it += 1;
  const int p = (int)(ctx->it & 1);
  // (SPLIT, N > 1: the scheduled merge of t-2 is waited on device by GATE_FWD's def_done flags)
  // N == 1: the prefetch copy (mark) runs on the side stream and nothing on
  // the main stream reads it (the prefetch check is a fingerprint, k_gate.cu)
  ctx->mark_pending = false;
  const int pre = ctx->prefetched ? 1 : 0;
  // N > 1 and prefetched: GATE_FWD also waits for sort(t) (computed one
  // iteration ahead), and the forward pulls each distinct row once (dedup)
  // using the sort's chunk descriptors; the coalesce then needs no sort gate.
  //   The gate does not wait for sort(t): it only records whether sort(t) is
  //   already complete (fwd_dd[p]); the forward dedups if so, else it gathers
  //   every token (identical Y).  Waiting would put the aux chain (push, tags,
  //   plan, sort) on the critical path when the sort is the slower side (LM).
  // (The forward's CTA 0 waiting for sort(t) instead of the GATE_SORTED
  // kernel measured GNMT -0.8 us, LM +2.9 us at N == 1 in round 1: a CTA
  // spinning in a wide kernel delays other streams' launches, §6 Liveness.)
  const int dedup = (pre && ctx->pl.N > 1 && ctx->fwd_dedupn) ? 1 : 0;
  // N == 1, prefetched: sort(t) was launched by backward(t-1) one step ago.
  // The forward takes a real stream dependency on it (an event join: a graph
  // edge when captured) instead of a GATE_SORTED spin kernel before the
  // coalesce — the coalesce is ordered after it through the forward.  A spin
  // in the forward's last CTA instead was measured to deadlock under CUDA
  // graphs (the graph may serialise the sort behind the spinning forward;
  // profiles/r02_tune), so no spin crosses a stream here.
  // (N > 1: the coalesce joins sort(t) instead — the forward must not wait for
  // the aux chain, whose sort follows a cross-GPU wait; see backward)
  const bool join = pre && ctx->pl.N == 1 && ctx->sort_join && ctx->sort_pending[p];
  if (join) CKC(ctx, cudaStreamWaitEvent(stream, ctx->ev_sorted[p], 0));
  ctx->fwd_joined = join;
  // N == 1 and joined: sort(t) is complete, so the forward may gather each
  // distinct row once per reduce chunk (SURVEY §8(f) NEXT-3 forward dedup)
  const int fdedup = (join && ctx->fwd_dedup1) ? 2 : dedup;
  CKC(ctx, gate(ctx, p, GATE_FWD, pre | (dedup << 1), stream));
  CKC(ctx, run_k(ctx, EMB_K_FWD, stream,
                 [&] { return launch_fwd(ctx->dc, ctx->lc, ids, n, out, p, pre, fdedup, stream); }));
  if (!pre) {
    // ids were not prefetched: sort them now on the auxiliary stream (the
    // forward pushed them; the sort publishes the push to the peers)
    CKC(ctx, cudaEventRecord(ctx->ev_main[p], stream));
    cudaStream_t sq = (ctx->pl.N == 1 && (p & 1)) ? ctx->aux2 : ctx->aux;
    if (sq == ctx->aux2) ctx->aux2_used = true;
    CKC(ctx, cudaStreamWaitEvent(sq, ctx->ev_main[p], 0));
    CKC(ctx, gate(ctx, p, GATE_SORT, 1 | 2 | 4, sq));
    CKC(ctx, run_k(ctx, EMB_K_SORT, sq, [&] {
      return launch_sort(ctx->dc, p, nullptr, 0, 0, ctx->pl.key64, ctx->pl.sort_smem, sq);
    }));
    CKC(ctx, cudaEventRecord(ctx->ev_sorted[p], sq));
    ctx->sort_pending[p] = true;
    ctx->aux_used = true;
  }
  ctx->prefetched = false;
  ctx->last_n = n;
  ctx->state = ST_AFTER_FWD;
  return EMB_OK;
}

emb_status emb_prefetch(emb_ctx* ctx, const int32_t* next_ids, int32_t n_next, emb_stream_t stream_) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (ctx->state == ST_AFTER_FWD || ctx->state == ST_CREATED || ctx->pf_armed) return EMB_ERR_STATE;
  if (!next_ids || n_next < 0) return EMB_ERR_INVALID_ARG;
  if (n_next > ctx->cfg.max_tokens) return EMB_ERR_CAPACITY;
  CKC(ctx, cudaEventRecord(ctx->ev_pre, reinterpret_cast<cudaStream_t>(stream_)));
  ctx->pf_ids = next_ids;
  ctx->pf_n = n_next;
  ctx->pf_armed = true;
  return EMB_OK;
}

#ifndef EMB_SORT_QUIET
#define EMB_SORT_QUIET 1  // N == 1 joined prefetch sorts skip the flag fences (see k_sort.cu)
#endif
emb_status emb_backward_exchange(emb_ctx* ctx, const void* grad_out, const int32_t* next_ids, int32_t n_next,
                                 emb_stream_t stream_) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (ctx->state != ST_AFTER_FWD) return EMB_ERR_STATE;
  if (ctx->last_n > 0 && !grad_out) return EMB_ERR_INVALID_ARG;
  if (next_ids && (n_next < 0 || n_next > ctx->cfg.max_tokens)) return EMB_ERR_CAPACITY;
  if (!next_ids) n_next = 0;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const int p = (int)(ctx->it & 1);
  const DevCtx& c = ctx->dc;
  const int mode = ctx->cfg.mode;
  const LaunchCfg& lc = ctx->lc;
  const int last_n = ctx->last_n;
  cudaStream_t side = ctx->side;
  cudaStream_t aux = ctx->aux;
  const int N = ctx->pl.N;
  const int do_mark = (mode == EMB_BWD_SPLIT && next_ids) ? 1 : 0;
  // Fork (not join): the aux / side streams are ordered after everything the
  // caller enqueued so far (next_ids / dY ready, forward(t) done).  An event
  // record on the main stream does not break its programmatic-launch chain; a
  // wait on the main stream would, so every join back into it is a device
  // flag gate instead (GATE_SORTED, GATE_MARKED, GATE_FWD's def_done).
  //   With emb_prefetch(next_ids) called before this step's forward, the fork
  //   point is that earlier position (the next batch's work overlaps forward(t)).
  const bool early = ctx->pf_armed && ctx->pf_ids == next_ids && ctx->pf_n == n_next && next_ids != nullptr;
  ctx->pf_armed = false;
  // The aux / side kernels of backward(t) take t from sorted[p] (the sort of t
  // precedes them on their stream) or the side stream's own count, never from
  // t_rec (written by forward(t), which an early fork may precede).
  // N > 1, sort(t) launched by backward(t-1) on aux: the coalesce below takes
  // a stream dependency on it (event join) instead of a GATE_SORTED kernel
  const bool sjoin = N > 1 && ctx->sort_join && ctx->sort_pending[p] && !ctx->fwd_joined;
  CKC(ctx, cudaEventRecord(ctx->ev_main[p], stream));
  cudaEvent_t fork = early ? ctx->ev_pre : ctx->ev_main[p];
  CKC(ctx, cudaStreamWaitEvent(aux, fork, 0));
  CKC(ctx, cudaStreamWaitEvent(side, fork, 0));
  ctx->aux_used = ctx->side_used = true;
  // the sort of this batch (aux stream) must be complete: a one-warp gate on a
  // device flag the sort sets (a host event here would break the PDL chain);
  // at N == 1 it also checks the prefetch fingerprints.  Enqueued before this
  // backward's aux / side work so that host launch order is also a valid
  // serial order (profilers replay kernels one at a time).
  // (N == 1 prefetched: the forward already joined the sort's event — the
  // coalesce checks the prefetch fingerprints in its CTA 0.)
  if (sjoin)
    CKC(ctx, cudaStreamWaitEvent(stream, ctx->ev_sorted[p], 0));
  else if (!ctx->fwd_joined)
    CKC(ctx, run_k(ctx, EMB_K_GATE, stream, [&] { return launch_gate(ctx->dc, p, GATE_SORTED, 0, stream); }));

  if (N == 1) {
    // N == 1: nothing on the critical path needs the D_next marks (the coalesce
    // applies every row), so
    //   aux:  a6 for the next batch straight from the caller's next_ids, one
    //         iteration ahead and first in line (the coalesce of t+1 waits for it);
    //   side: a5 (ids copy for the forward's prefetch check + D_next marks) and
    //         the a8 slot tables of this batch.
    // next_ids is read asynchronously until the next backward (header contract).
    if (next_ids) {
      // the sort of t+1 goes to the stream of its parity: consecutive sorts may
      // overlap (each is one 8-SM cluster), so the sort no longer bounds the step
      cudaStream_t sq = ((p ^ 1) & 1) ? ctx->aux2 : aux;
      if (sq == ctx->aux2) ctx->aux2_used = true;
      CKC(ctx, cudaStreamWaitEvent(sq, fork, 0));
      if (ctx->tables_pending[p ^ 1]) CKC(ctx, cudaStreamWaitEvent(sq, ctx->ev_tables[p ^ 1], 0));
      CKC(ctx, run_k(ctx, EMB_K_SORT, sq, [&] {
        return launch_sort(c, p ^ 1, next_ids, n_next, ctx->sort_join && EMB_SORT_QUIET ? 3 : 2, ctx->pl.key64,
                           ctx->pl.sort_smem, sq);
      }));
      CKC(ctx, cudaEventRecord(ctx->ev_sorted[p ^ 1], sq));
      ctx->sort_pending[p ^ 1] = true;
      ctx->tables_pending[p ^ 1] = false;
    }
    // tables(t) reads sort(t)'s unique lists: an event join from aux into side
    // (joins into side do not touch the main stream's programmatic chain; a
    // spinning side gate started before the forward was observed to hold back
    // the main stream's launches — timeouts)
    if (ctx->sort_pending[p]) CKC(ctx, cudaStreamWaitEvent(side, ctx->ev_sorted[p], 0));
    CKC(ctx, run_k(ctx, EMB_K_ROUTE, side, [&] { return launch_markpush(c, p, next_ids, n_next, 1, side); }));
    CKC(ctx, run_k(ctx, EMB_K_ROUTE, side, [&] { return launch_marktag(c, p, do_mark, 1, 1, side); }));
    CKC(ctx, cudaEventRecord(ctx->ev_marked, side));
    ctx->mark_pending = true;
    CKC(ctx, run_k(ctx, EMB_K_TABLES, side, [&] { return launch_tables(c, p, 1, side); }));
    CKC(ctx, cudaEventRecord(ctx->ev_tables[p], side));
    ctx->tables_pending[p] = true;
    ctx->side_used = true;
    ctx->aux_used = true;
  } else {
    // a5 on the aux stream: the prefetch push of ids(t+1) and the D_next tags
    // overlap the segmented reduce (which does not need them); only the apply,
    // which routes prior vs scheduled rows, waits for them (GATE_MARKED).
    // aux chain (critical at N > 1: the forward of t+1 dedups with sort(t+1)):
    // push ids(t+1) -> one gate (publish + wait ids(t+1), and this rank's
    // scheduled push of t-1 past the routing tables) -> D_next tags -> merge
    // plan -> sort(t+1) -> the Alg. 1 tables of t (presentation, last).
    // next_ids == NULL (D_next = ∅): nothing is pushed or published for batch
    // t+1 here — forward(t+1) pushes, publishes and sorts its own ids — so the
    // gate only keeps the wait that frees parity p's tags / plan (flag 8)
    // (sort stream aux2: the aux chain reads sort(t)'s lists and epoch, so it
    // first joins sort(t); the sort of t+1 forks from aux right after the gate)
    const bool s2 = ctx->aux2 != nullptr;
    if (s2 && ctx->sort_pending[p]) CKC(ctx, cudaStreamWaitEvent(aux, ctx->ev_sorted[p], 0));
    if (next_ids) CKC(ctx, run_k(ctx, EMB_K_ROUTE, aux, [&] { return launch_markpush(c, p, next_ids, n_next, 0, aux); }));
    CKC(ctx, gate(ctx, p ^ 1, GATE_SORT, next_ids ? (1 | 2 | 4 | 8 | 16) : (8 | 16), aux));
    if (next_ids && s2) {
      CKC(ctx, cudaEventRecord(ctx->ev_gsort, aux));
      CKC(ctx, cudaStreamWaitEvent(ctx->aux2, ctx->ev_gsort, 0));
      ctx->aux2_used = true;
      CKC(ctx, run_k(ctx, EMB_K_SORT, ctx->aux2, [&] {
        return launch_sort(c, p ^ 1, nullptr, 0, 1, ctx->pl.key64, ctx->pl.sort_smem, ctx->aux2);
      }));
      CKC(ctx, cudaEventRecord(ctx->ev_sorted[p ^ 1], ctx->aux2));
      ctx->sort_pending[p ^ 1] = true;
    }
    CKC(ctx, run_k(ctx, EMB_K_ROUTE, aux, [&] { return launch_marktag(c, p, do_mark, 0, 0, aux); }));
    CKC(ctx, cudaEventRecord(ctx->ev_plan[p], aux));  // D_next tags of t+1 complete (the apply routes by them)
    CKC(ctx, run_k(ctx, EMB_K_ROUTE, aux, [&] { return launch_plan(c, p, aux); }));
    ctx->aux_used = true;
    if (next_ids && !s2) {
      CKC(ctx, run_k(ctx, EMB_K_SORT, aux, [&] {
        return launch_sort(c, p ^ 1, nullptr, 0, 1, ctx->pl.key64, ctx->pl.sort_smem, aux);
      }));
      CKC(ctx, cudaEventRecord(ctx->ev_sorted[p ^ 1], aux));
      ctx->sort_pending[p ^ 1] = true;
    }
    // the Alg. 1 slot tables of t (presentation: stats / debug) stay off the
    // aux chain in SPLIT (side stream, after the scheduled push: see below)
    if (mode != EMB_BWD_SPLIT) CKC(ctx, run_k(ctx, EMB_K_TABLES, aux, [&] { return launch_tables(c, p, 0, aux); }));
  }
  ctx->sort_pending[p] = false;
  if (mode == EMB_BWD_RAW) {
    CKC(ctx, run_k(ctx, EMB_K_RAWPUSH, stream, [&] { return launch_rawpush(c, lc, grad_out, last_n, p, stream); }));
    CKC(ctx, gate(ctx, p, GATE_PUB0, 0, stream));
    CKC(ctx, run_k(ctx, EMB_K_RAWCOAL, stream, [&] { return launch_rawcoal(c, lc, p, stream); }));
    CKC(ctx, run_k(ctx, EMB_K_MERGE0, stream, [&] { return launch_merge(c, lc, p, 0, stream); }));
  } else {
    // (SPLIT, N > 1: the D_next tags of t+1 must be complete before the apply
    // routes rows; a one-warp gate, not the reduce kernel's CTA 0: a wide
    // kernel spinning on a flag was observed to hold back the launch of the
    // aux-stream kernel that sets it — timeouts)
    const int cg = (N == 1 ? 1 : 0);
    CKC(ctx, run_k(ctx, EMB_K_COAL, stream, [&] { return launch_coal(c, lc, grad_out, p, cg, stream); }));
    // N > 1 SPLIT: the apply routes by the D_next tags of t+1 (aux, launched
    // above in this call): an event join, or the GATE_MARKED spin kernel
    if (mode == EMB_BWD_SPLIT && N > 1) {
      if (ctx->sort_join) CKC(ctx, cudaStreamWaitEvent(stream, ctx->ev_plan[p], 0));
      else CKC(ctx, gate(ctx, p, GATE_MARKED, 0, stream));
    }
    CKC(ctx, run_k(ctx, EMB_K_APPLY, stream, [&] { return launch_coal_apply(c, lc, grad_out, p, stream); }));
    // N == 1: the coalesce applied every row's update itself (one source = the
    // merged gradient); there is nothing to exchange or merge, for either part.
    if (mode == EMB_BWD_SPLIT && ctx->pl.N > 1) CKC(ctx, cudaEventRecord(ctx->ev_prior[p], stream));  // apply done
    if (ctx->pl.N > 1) {
      CKC(ctx, gate(ctx, p, GATE_PUB0, 0, stream));
      CKC(ctx, run_k(ctx, EMB_K_MERGE0, stream, [&] { return launch_merge(c, lc, p, 0, stream); }));
    }
    if (mode == EMB_BWD_SPLIT && ctx->pl.N > 1) {
      // scheduled part: lowest-priority side stream, once the apply of t staged
      // the scheduled rows: an event recorded on the main stream after the
      // apply (a record does not break the main stream's PDL chain)
      CKC(ctx, cudaStreamWaitEvent(side, ctx->ev_prior[p], 0));
      if (ctx->pl.N > 1)  // N == 1: coal wrote every row to its receive slot directly
        CKC(ctx, run_k(ctx, EMB_K_DEFPUSH, side, [&] { return launch_defpush(c, lc, p, side); }));
      // tables(t) reads sort(t)'s unique lists and the D_next tags of t+1 (both
      // complete: the apply joined them); GATE_PUB1 then records SEQ_DEFPUSHED,
      // which the sort of t+2 waits for before it rewrites the lists
      CKC(ctx, run_k(ctx, EMB_K_TABLES, side, [&] { return launch_tables(c, p, 0, side); }));
      CKC(ctx, gate(ctx, p, GATE_PUB1, 0, side));
      CKC(ctx, run_k(ctx, EMB_K_MERGE1, side, [&] { return launch_merge(c, lc, p, 1, side); }));
      CKC(ctx, gate(ctx, p, GATE_DEFDONE, 0, side));  // def_done(t) to every owner
      ctx->side_used = true;
    }
  }
  ctx->prefetched = next_ids != nullptr;
  ctx->bwd_done += 1;
  ctx->state = ST_READY;
  return EMB_OK;
}

emb_status dense_allreduce_enqueue(emb_ctx* ctx, void* buf, int64_t count, emb_dtype dtype, int32_t priority,
                                   emb_event_t ready, int64_t* ticket) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (!ctx->dq) return EMB_ERR_STATE;
  if (!buf || count < 0 || !ticket || (dtype != EMB_FP32 && dtype != EMB_BF16)) return EMB_ERR_INVALID_ARG;
  st = dense_queue_enqueue(ctx->dq, buf, count, dtype, priority, reinterpret_cast<cudaEvent_t>(ready), ticket);
  if (st == EMB_ERR_CUDA || st == EMB_ERR_NCCL) ctx->poisoned = st;
  return st;
}

emb_status dense_queue_flush(emb_ctx* ctx) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (!ctx->dq) return EMB_OK;
  st = dense_queue_flush_all(ctx->dq);
  if (st == EMB_ERR_CUDA || st == EMB_ERR_NCCL) ctx->poisoned = st;
  return st;
}

emb_status dense_wait(emb_ctx* ctx, int64_t ticket, emb_stream_t consumer) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (!ctx->dq) return EMB_ERR_STATE;
  return dense_queue_wait(ctx->dq, ticket, reinterpret_cast<cudaStream_t>(consumer));
}

static emb_status sticky_err(emb_ctx* ctx) {
  int err = 0;
  CKC(ctx, cudaMemcpy(&err, ctx->dc.err, 4, cudaMemcpyDeviceToHost));
  if (err & ERR_ID) return EMB_ERR_ID_RANGE;
  if (err & ERR_STATE) return EMB_ERR_STATE;
  if (err & ERR_TIMEOUT) return EMB_ERR_TIMEOUT;
  return EMB_OK;
}

emb_status emb_flush(emb_ctx* ctx, emb_stream_t stream_) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  CKC(ctx, cudaSetDevice(ctx->cfg.device));
  st = emb_join(ctx, stream_);
  if (st != EMB_OK) return st;
  if (ctx->dq) {
    st = dense_queue_flush_all(ctx->dq);
    if (st != EMB_OK) { ctx->poisoned = st; return st; }
    st = dense_queue_wait_all(ctx->dq, stream);
    if (st != EMB_OK) { ctx->poisoned = st; return st; }
  }
  CKC(ctx, cudaStreamSynchronize(stream));
  return sticky_err(ctx);
}

emb_status emb_join(emb_ctx* ctx, emb_stream_t stream_) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  // everything enqueued so far on the library's streams precedes later work on `stream`
  if (ctx->aux_used) {
    CKC(ctx, cudaEventRecord(ctx->ev_join_aux, ctx->aux));
    CKC(ctx, cudaStreamWaitEvent(stream, ctx->ev_join_aux, 0));
    ctx->aux_used = false;
  }
  if (ctx->aux2_used) {
    CKC(ctx, cudaEventRecord(ctx->ev_join_aux2, ctx->aux2));
    CKC(ctx, cudaStreamWaitEvent(stream, ctx->ev_join_aux2, 0));
    ctx->aux2_used = false;
  }
  if (ctx->side_used) {
    CKC(ctx, cudaEventRecord(ctx->ev_join_side, ctx->side));
    CKC(ctx, cudaStreamWaitEvent(stream, ctx->ev_join_side, 0));
    ctx->side_used = false;
  }
  for (int p = 0; p < 2; ++p) {
    ctx->def_pending[p] = false;
    ctx->sort_pending[p] = false;
    ctx->tables_pending[p] = false;
  }
  ctx->mark_pending = false;
  return EMB_OK;
}

emb_status emb_profile(emb_ctx* ctx, int32_t enable) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  ctx->prof = enable != 0;
  return EMB_OK;
}

emb_status emb_profile_read(emb_ctx* ctx, double* ms, int64_t* count) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (!ms || !count) return EMB_ERR_INVALID_ARG;
  CKC(ctx, cudaSetDevice(ctx->cfg.device));
  CKC(ctx, cudaDeviceSynchronize());
  for (int k = 0; k < EMB_NUM_KERNELS; ++k) { ms[k] = 0.0; count[k] = 0; }
  // EMB_PROF_TIMELINE=<file>: append "kind start_us dur_us" per launch (debug aid)
  FILE* tl = nullptr;
  if (const char* tp = getenv("EMB_PROF_TIMELINE")) {
    char path[512];
    snprintf(path, sizeof path, "%s.%d", tp, ctx->cfg.rank);
    tl = fopen(path, "a");
  }
  for (auto& r : ctx->prof_recs) {
    float t = 0.f;
    if (tl) {
      float t0 = 0.f, d = 0.f;
      cudaEventElapsedTime(&t0, ctx->prof_recs.front().a, r.a);
      cudaEventElapsedTime(&d, r.a, r.b);
      fprintf(tl, "%d %.2f %.2f\n", r.kind, t0 * 1e3f, d * 1e3f);
    }
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) {
      ms[r.kind] += t;
      count[r.kind] += 1;
    }
  }
  for (auto& r : ctx->prof_recs) {  // after the loop: the timeline measures from the first event
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  if (tl) fclose(tl);
  ctx->prof_recs.clear();
  return EMB_OK;
}

emb_status emb_get_stats(emb_ctx* ctx, emb_stats* out) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (!out) return EMB_ERR_INVALID_ARG;
  CKC(ctx, cudaSetDevice(ctx->cfg.device));
  CKC(ctx, cudaDeviceSynchronize());
  memset(out, 0, sizeof(*out));
  const int N = ctx->pl.N;
  out->iter = ctx->bwd_done;
  out->world = N;
  if (ctx->bwd_done > 0) {
    const int p = (int)(ctx->it & 1);
    std::vector<int> cnt(N * CNT_W);
    CKC(ctx, cudaMemcpy(cnt.data(), ctx->dc.counts + (size_t)p * N * CNT_W, N * CNT_W * 4, cudaMemcpyDeviceToHost));
    for (int n = 0; n < N; ++n) {
      out->n_tokens[n] = cnt[n * CNT_W + CNT_T];
      out->u[n] = cnt[n * CNT_W + CNT_U];
      out->p[n] = cnt[n * CNT_W + CNT_P];
      out->q[n] = cnt[n * CNT_W + CNT_U] - cnt[n * CNT_W + CNT_P];
    }
  }
  std::vector<unsigned long long> s(3 * N);
  CKC(ctx, cudaMemcpy(s.data(), ctx->dc.stats, 3 * N * 8, cudaMemcpyDeviceToHost));
  for (int n = 0; n < N; ++n) {
    out->fwd_bytes_pulled[n] = (int64_t)s[n];
    out->bwd_bytes_pushed[n] = (int64_t)s[N + n];
    out->ids_bytes_pushed[n] = (int64_t)s[2 * N + n];
  }
  CKC(ctx, cudaMemcpy(&out->err_flags, ctx->dc.err, 4, cudaMemcpyDeviceToHost));
  out->kernel_launches = ctx->launches;
  return EMB_OK;
}

emb_status emb_debug_copy(emb_ctx* ctx, int32_t item, int32_t src, void* host, size_t cap, size_t* n) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (!n || (!host && cap)) return EMB_ERR_INVALID_ARG;
  const int N = ctx->pl.N;
  *n = 0;
  CKC(ctx, cudaSetDevice(ctx->cfg.device));
  CKC(ctx, cudaDeviceSynchronize());
  if (item == EMB_DBG_ERRINFO) {
    *n = 32;
    if (cap < 32 * 4) return EMB_ERR_CAPACITY;
    CKC(ctx, cudaMemcpy(host, ctx->dc.err_info, 32 * 4, cudaMemcpyDeviceToHost));
    return EMB_OK;
  }
  if (item == EMB_DBG_TIMESTAMPS) {
    *n = EMB_TRACE_SLOTS;
    if (cap < EMB_TRACE_SLOTS * 8) return EMB_ERR_CAPACITY;
    CKC(ctx, cudaMemcpy(host, ctx->dc.dbg_ts, EMB_TRACE_SLOTS * 8, cudaMemcpyDeviceToHost));
    return EMB_OK;
  }
  if (item == EMB_DBG_ISSUE_LOG) {
    std::vector<int64_t> log;
    if (ctx->dq) dense_queue_issue_log(ctx->dq, &log);
    *n = log.size();
    if (cap < log.size() * 8) return EMB_ERR_CAPACITY;
    if (!log.empty()) memcpy(host, log.data(), log.size() * 8);
    return EMB_OK;
  }
  if (ctx->bwd_done == 0) return EMB_ERR_STATE;
  const int p = (int)(ctx->it & 1);
  if (item == EMB_DBG_COUNTS) {
    *n = (size_t)N * 4;
    if (cap < *n * 4) return EMB_ERR_CAPACITY;
    std::vector<int> all(N * CNT_W);
    CKC(ctx, cudaMemcpy(all.data(), ctx->dc.counts + (size_t)p * N * CNT_W, N * CNT_W * 4, cudaMemcpyDeviceToHost));
    int* h = static_cast<int*>(host);
    for (int q = 0; q < N; ++q)
      for (int j = 0; j < 4; ++j) h[q * 4 + j] = all[q * CNT_W + j];
    return EMB_OK;
  }
  if (src < 0 || src >= N) return EMB_ERR_INVALID_ARG;
  int cnt[CNT_W];
  CKC(ctx, cudaMemcpy(cnt, ctx->dc.counts + ((size_t)p * N + src) * CNT_W, CNT_W * 4, cudaMemcpyDeviceToHost));
  const int* dptr = nullptr;
  size_t len = 0;
  const size_t off = ((size_t)p * N + src) * ctx->cfg.max_tokens;
  switch (item) {
    case EMB_DBG_GIDS:
      dptr = reinterpret_cast<const int*>(ctx->sym + ctx->pl.lay.gids) + off;
      len = cnt[0];
      break;
    case EMB_DBG_SLOT_IDS: dptr = ctx->dc.slot_id + off; len = cnt[1]; break;
    case EMB_DBG_PERM: dptr = ctx->dc.perm + off; len = cnt[0]; break;
    default: return EMB_ERR_INVALID_ARG;
  }
  *n = len;
  if (cap < len * 4) return EMB_ERR_CAPACITY;
  if (len) CKC(ctx, cudaMemcpy(host, dptr, len * 4, cudaMemcpyDeviceToHost));
  return EMB_OK;
}

emb_status emb_state_ptr(emb_ctx* ctx, int32_t item, void** ptr) {
  emb_status st = ctx_check(ctx);
  if (st != EMB_OK) return st;
  if (!ptr) return EMB_ERR_INVALID_ARG;
  switch (item) {
    case EMB_STATE_SHARD: *ptr = ctx->sym + ctx->pl.lay.shard; return EMB_OK;
    case EMB_STATE_ADAM_M: *ptr = ctx->dc.adam_m; return ctx->dc.adam_m ? EMB_OK : EMB_ERR_STATE;
    case EMB_STATE_ADAM_V: *ptr = ctx->dc.adam_v; return ctx->dc.adam_v ? EMB_OK : EMB_ERR_STATE;
  }
  return EMB_ERR_INVALID_ARG;
}

emb_status emb_queue_issue_order(const int32_t* priorities, int32_t n, int32_t window, int32_t* out) {
  if (n < 0 || window < 1 || (n > 0 && (!priorities || !out))) return EMB_ERR_INVALID_ARG;
  std::vector<int64_t> order;
  issue_rule_order(priorities, n, window, &order);
  for (int i = 0; i < n; ++i) out[i] = (int32_t)order[i];
  return EMB_OK;
}

emb_status emb_shard_destroy(emb_ctx* ctx) {
  if (!ctx) return EMB_ERR_INVALID_ARG;
  cudaSetDevice(ctx->cfg.device);
  cudaDeviceSynchronize();
  if (ctx->dq) dense_queue_destroy(ctx->dq);
  for (int s = 0; s < EMB_MAX_WORLD; ++s)
    if (ctx->peer_open[s]) cudaIpcCloseMemHandle(ctx->dc.sym[s]);
  for (void* p : ctx->allocs) cudaFree(p);
  if (ctx->sym) cudaFree(ctx->sym);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->aux2) cudaStreamDestroy(ctx->aux2);
  for (int i = 0; i < 2; ++i) {
    if (ctx->ev_prior[i]) cudaEventDestroy(ctx->ev_prior[i]);
    if (ctx->ev_def[i]) cudaEventDestroy(ctx->ev_def[i]);
    if (ctx->ev_main[i]) cudaEventDestroy(ctx->ev_main[i]);
    if (ctx->ev_sorted[i]) cudaEventDestroy(ctx->ev_sorted[i]);
    if (ctx->ev_tables[i]) cudaEventDestroy(ctx->ev_tables[i]);
    if (ctx->ev_plan[i]) cudaEventDestroy(ctx->ev_plan[i]);
  }
  for (cudaEvent_t e : {ctx->ev_marked, ctx->ev_join_aux, ctx->ev_join_side, ctx->ev_pre, ctx->ev_join_aux2,
                        ctx->ev_gsort}) {
    if (e) cudaEventDestroy(e);
  }
  delete ctx;
  return EMB_OK;
}

}  // extern "C"
