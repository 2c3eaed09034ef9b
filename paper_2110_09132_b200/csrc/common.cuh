// common.cuh — device-side layout, context and primitives shared by the
// EmbRace exchange kernels (sm_100a).  Product code: never includes or links
// anything from oracle/.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#define EMB_WMAX 8

namespace emb {

enum Mode { RAW = 0, COAL = 1, SPLIT = 2 };
enum Optim { SGD = 0, ADAM = 1, ADAGRAD = 2 };
enum DType { F32 = 0, BF16 = 1 };
enum ErrBit { ERR_ID = 1, ERR_STATE = 2, ERR_TIMEOUT = 4 };
// counts[p][n][CNT_W]
//   written by sort(t):   T, U (unique kept ids), NCH (reduce chunks), NLONG (multi-chunk uniques)
//   written by tables(t): P (prior uniques of the Alg. 1 split; stats / debug only)
// chunk_desc[].w = chunks of the unique | (first position + 1) << DESC_POS_SHIFT for
// a single-row unique (its one position rides with the descriptor: the reduce
// needs no perm load for it), 0 above the chunk count otherwise
constexpr int DESC_POS_SHIFT = 13;
constexpr int DESC_NCH_MASK = (1 << DESC_POS_SHIFT) - 1;
__host__ __device__ __forceinline__ int desc_nch(int w) { return w & DESC_NCH_MASK; }
__host__ __device__ __forceinline__ int desc_pos1(int w) { return (w >> DESC_POS_SHIFT) - 1; }
enum CountSlot { CNT_T = 0, CNT_U = 1, CNT_P = 2, CNT_NCH = 3, CNT_NLONG = 4, CNT_W = 8 };

// Peer-written flags living in every rank's NVLink-visible region.  Slot [n]
// is written only by rank n (epoch values = iteration number t, monotone).
struct Flags {
  uint32_t ids[EMB_WMAX];         // ids of iteration v are in my gids[v&1][n]
  uint32_t pub[2][EMB_WMAX];      // part 0 (prior / all) / part 1 (scheduled) rows of iteration v
                                  // from sender n are in my recv[v&1][n]
  uint32_t prior_done[EMB_WMAX];  // owner n applied the prior part of iteration v
  uint32_t def_done[EMB_WMAX];    // owner n applied the scheduled part of iteration v
  uint32_t boot[EMB_WMAX];        // rank n finished emb_shard_init (its shard is loaded)
  uint32_t pad[64 - 6 * EMB_WMAX];
};

// Byte offsets inside the symmetric (IPC-exported) region; identical on every rank.
struct SymLayout {
  size_t shard;   // [L][d]             table dtype     (peers read: forward pull)
  size_t gids;    // [2][N][max_tok]    int32           (peers write: id all-gather)
  size_t ntok;    // [2][N]             int32
  size_t recv;    // [2][N][max_tok][d] wire = table dtype (senders write: grad AlltoAll),
                  //                    row i = sender's unique id i
  size_t flags;   // Flags
  size_t total;
};

// Everything a kernel needs, passed by value.
struct DevCtx {
  int N, r;
  long long L;
  int D, d, esz;          // esz: bytes per element of the table dtype
  int dtype, mode, optim;
  int max_tok;
  int bypass;             // EMB_SINGLE_BYPASS: single-row uniques skip coal_reduce (apply reads dY)
  int pdl_early;          // EMB_PDL_EARLY: compute kernels trigger their dependents right after griddepcontrol.wait
  int cpr, cps;           // 16-byte chunks per full row (D*esz/16) / per column slice (d*esz/16)
  long long pad_id;
  float lr, beta1, beta2, eps, scale;
  unsigned long long timeout_ns;
  int C;                  // rows per reduce chunk
  int max_chunks;         // per source per parity
  int max_long;           // multi-chunk uniques per source per parity (<= max_tok / (C+1) + 1)
  int idbits, posbits;

  char* sym[EMB_WMAX];    // base of every rank's symmetric region (own included)
  SymLayout lay;

  // local (not peer-visible); [2] = iteration parity p = t & 1
  float* adam_m;          // [L][d]   Adam first moment; Adagrad: the squared-gradient accumulator
  float* adam_v;          // [L][d]
  int* nextmark;          // [2][L]   epoch tag: id in D_next of iteration v <=> nextmark[v&1][id] == v+1
  unsigned long long* slotmap;  // [2][L][N] (t << 32) | i — source n holds id as unique i at iteration t (N > 1)
  int* perm;              // [2][N][max_tok]    positions sorted by (dropped, id, position)
  int* uid;               // [2][N][max_tok]    ascending unique kept ids
  int* upos;              // [2][N][max_tok]    single-row unique -> its position, else -1
  int* useg;              // [2][N][max_tok+1]  unique i -> first index into perm (useg[U] = end)
  int* chunk_off;         // [2][N][max_tok+1]  unique i -> first reduce chunk
  int4* chunk_desc;       // [2][N][max_chunks] chunk -> {unique i, perm begin, perm end, chunks of i}
  int* long_u;            // [2][N][max_long]   uniques with more than one chunk
  int* slot_id;           // [2][N][max_tok]    Alg. 1 slot order (prior asc, then scheduled asc) — tables
  int* plan;              // [2][2 parts][N*max_tok][1+N] owner merge plan: id, then the unique index of
                          //   the id at every source (-1: absent); one entry per distinct id (N > 1)
  int* plan_cnt;          // [2][2]  entries per part
  int* counts;            // [2][N][CNT_W]
  float* scratch;         // [2][N][max_chunks][dw] chunk partials (dw = D sender / d RAW owner)
  float* gcoal;           // [max_tok][D] fp32  sender-coalesced rows of single-chunk uniques (COAL/SPLIT)
  char* stage;            // [2][max_tok][D]    scheduled coalesced rows waiting to be pushed (N > 1)
  float* gc_owner;        // [2][N][max_tok][d] RAW: owner-coalesced rows (fp32)
  unsigned int* t_rec;    // [2]   t of the iteration using parity p
  unsigned int* sorted;   // [2]   t of the last completed sort of parity p (gate before the coalesce)
  unsigned int* sort_cnt; // [2]   clusters of the running sort that finished (re-armed by the last)
  unsigned int* sort_count; // [2] completed sorts of parity p (one per iteration: ceil(t/2) after t)
  unsigned int* side_it;  // [1]   N == 1: backward calls seen by the side stream (its iteration number)
  unsigned int* marked;   // [2]   t of the last completed mark (prefetch push + D_next tags) of parity p
  unsigned int* mark_cnt; // [2]   CTAs of the running mark that finished (re-armed by the last)
  unsigned int* seq;      // [4]   progress records: [SEQ_BWD] t past the sort gate, [SEQ_APPLIED] t past the
                          //       apply, [SEQ_DEFPUSHED] t past the scheduled push (the sort of t+2 waits it)
  unsigned int* fwd_dd;   // [2]   N > 1: the forward of parity p dedups (sort(t) was already complete at its gate)
  unsigned int* merge_cnt;  // [2] N > 1: CTAs of the running merge(part 0) of parity p that finished
  unsigned int* fp;       // [2][4] N == 1 prefetch check: {sum h(ids fwd), n fwd, sum h(next_ids sort), n sort}
  float* alpha;           // [2]   Adam step size alpha_t (computed once by the forward)
  int* err;               // sticky error bits
  unsigned* err_info;     // [8][4] + count: expired waits (site, observed, target, set)
  unsigned long long* stats;  // [3][N] bytes: fwd pulled / bwd pushed / ids pushed
  unsigned long long* dbg_ts; // [EMB_TRACE_SLOTS] kernel trace (EMB_TRACE builds only)
};

// Kernel trace (EMB_TRACE builds only; a debug aid, compiled out otherwise):
// dbg_ts[(t & 15)][EMB_TRACE_KINDS][8] globaltimer stamps — 0: block 0 entered (before
// the PDL wait), 1: block 0 past its dependency/flag waits, 2: last block
// finished (max over blocks), 3..7: block 0 at kernel-specific points
// (EMB_TR_AT).  Read with emb_debug_copy(EMB_DBG_TIMESTAMPS).
#define EMB_TRACE_KINDS 20
#define EMB_TRACE_SLOTS (16 * EMB_TRACE_KINDS * 8)
#ifdef EMB_TRACE
#define EMB_TR_IDX(kind, t, slot) (((((t)&15) * EMB_TRACE_KINDS) + (kind)) * 8 + (slot))
#define EMB_TR_ENTRY() const unsigned long long tr_entry_ = globaltimer()
#define EMB_TR_BEGIN(kind, t)                                                             \
  do {                                                                                    \
    if (blockIdx.x == 0 && threadIdx.x == 0) c.dbg_ts[EMB_TR_IDX(kind, t, 0)] = tr_entry_; \
  } while (0)
#define EMB_TR_AT(kind, t, slot)                                                              \
  do {                                                                                        \
    if (blockIdx.x == 0 && threadIdx.x == 0) c.dbg_ts[EMB_TR_IDX(kind, t, slot)] = globaltimer(); \
  } while (0)
#define EMB_TR_END(kind, t)                                                              \
  do {                                                                                   \
    if (threadIdx.x == 0) atomicMax(c.dbg_ts + EMB_TR_IDX(kind, t, 2), globaltimer());   \
  } while (0)
#else
#define EMB_TR_ENTRY() do {} while (0)
#define EMB_TR_BEGIN(kind, t) do {} while (0)
#define EMB_TR_AT(kind, t, slot) do {} while (0)
#define EMB_TR_END(kind, t) do {} while (0)
#endif
#define EMB_TR_WAITED(kind, t) EMB_TR_AT(kind, t, 1)
#define EMB_TR_MID(kind, t) EMB_TR_AT(kind, t, 3)

// ----------------------------------------------------------------- addressing
__device__ __forceinline__ char* shard_of(const DevCtx& c, int s) { return c.sym[s] + c.lay.shard; }
__device__ __forceinline__ int* gids_of(const DevCtx& c, int s, int p, int n) {
  return reinterpret_cast<int*>(c.sym[s] + c.lay.gids) + ((size_t)(p * c.N + n)) * c.max_tok;
}
__device__ __forceinline__ int* ntok_of(const DevCtx& c, int s, int p, int n) {
  return reinterpret_cast<int*>(c.sym[s] + c.lay.ntok) + p * c.N + n;
}
__device__ __forceinline__ char* recv_of(const DevCtx& c, int s, int p, int n) {
  return c.sym[s] + c.lay.recv + ((size_t)(p * c.N + n)) * c.max_tok * (size_t)c.d * c.esz;
}
__device__ __forceinline__ Flags* flags_of(const DevCtx& c, int s) {
  return reinterpret_cast<Flags*>(c.sym[s] + c.lay.flags);
}
__device__ __forceinline__ size_t pn(const DevCtx& c, int p, int n) { return (size_t)(p * c.N + n); }
__device__ __forceinline__ const int* counts_of(const DevCtx& c, int p, int n) {
  return c.counts + pn(c, p, n) * CNT_W;
}
// Alg. 1 class of an id in iteration t (parity p): prior iff in the gathered next batch
__device__ __forceinline__ bool is_prior(const DevCtx& c, int p, uint32_t t, int id) {
  return c.mode != SPLIT || __ldcg(c.nextmark + (size_t)p * c.L + id) == (int)(t + 1);
}

// Position-hashed id for the N == 1 prefetch check: the sums over a batch of
// h(id, j) computed by the forward (ids of t) and by the sort (next_ids given
// at t-1) must agree (a mismatch is missed with probability ~2^-32).
__device__ __forceinline__ unsigned prefetch_hash(int id, int j) {
  unsigned x = (unsigned)id * 0x9E3779B1u ^ ((unsigned)j * 0x85EBCA77u + 0x165667B1u);
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  x ^= x >> 12;
  return x;
}

// ----------------------------------------------------------------- memory model
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Message-passing release at system scope: acq_rel (not sc) is what the
// data -> flag pattern needs; it is cumulative over what this thread observed
// (the completed producer grid after griddepcontrol.wait, or its CTA's stores
// after __syncthreads).
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until *flag >= target (epoch compare, wrap-safe) or the bound expires.
// On expiry: sticky ERR_TIMEOUT, and the first expired wait is described in
// err_info = {site, observed value, target, 1} (emb_debug_copy EMB_DBG_ERRINFO).
__device__ __forceinline__ void note_timeout(const DevCtx& c, int site, uint32_t seen, uint32_t target) {
  atomicOr(c.err, ERR_TIMEOUT);
  // up to 8 expired waits, in expiry order: {site, seen, target, 1}
  const unsigned slot = atomicAdd(c.err_info + 32, 1u);
  if (slot < 8) {
    c.err_info[slot * 4 + 0] = (unsigned)site;
    c.err_info[slot * 4 + 1] = seen;
    c.err_info[slot * 4 + 2] = target;
    c.err_info[slot * 4 + 3] = 1u;
  }
}
__device__ __forceinline__ void wait_flag(const DevCtx& c, const uint32_t* flag, uint32_t target, int site = 0) {
  if ((int)(ld_acquire_sys(flag) - target) >= 0) return;
  unsigned long long t0 = globaltimer();
  uint32_t v;
  while ((int)((v = ld_acquire_sys(flag)) - target) < 0) {
    __nanosleep(32);
    if (globaltimer() - t0 > c.timeout_ns) {
      note_timeout(c, site, v, target);
      return;
    }
  }
}

// spin (bounded) until a local epoch flag reaches t
__device__ __forceinline__ void wait_local(const DevCtx& c, const uint32_t* flag, uint32_t t, int site) {
  const unsigned long long t0 = globaltimer();
  uint32_t v;
  while ((int)((v = ld_acquire_gpu(flag)) - t) < 0) {
    __nanosleep(32);
    if (globaltimer() - t0 > c.timeout_ns) {
      note_timeout(c, site, v, t);
      return;
    }
  }
}

// N == 1: every producer/consumer pair is ordered by the stream or an event,
// so the flag protocol (and its system fences) is skipped entirely.
__device__ __forceinline__ void wait_all(const DevCtx& c, const uint32_t* flags, uint32_t target, int site = 0) {
  if (c.N == 1) return;
  for (int s = 0; s < c.N; ++s) wait_flag(c, flags + s, target, site * 16 + s);
}

// Publish value v into slot [c.r] of field `field` (an offset into Flags) of
// every rank's flags.  Called by ONE thread of the kernel that follows the
// producer, after griddepcontrol.wait (same stream) or a full graph/event
// dependency (other stream): the producer grid has completed and its stores
// are visible to this thread.  One fence.acq_rel.sys then orders everything
// this thread has observed (cumulativity: the producer grid's local and peer
// stores) before the flag stores at system scope, so a peer that reads the
// flag with ld.acquire.sys sees the data — the PTX message-passing pattern,
// without relying on an end-of-grid flush that the memory model does not
// state.  (Round 1 used relaxed flag stores with no fence: a fence.sc.sys per
// publish had cost 2-7 us under concurrent NVLink traffic, kernel trace
// profiles/r01_trace_n2.txt; the build flag EMB_RELAXED_PUBLISH restores that
// variant for measurement only.)  Stores made by the SAME kernel before a
// flag (mark) take fence_acq_rel_sys() themselves.
__device__ __forceinline__ void publish2(const DevCtx& c, size_t off_a, uint32_t va, bool do_a, size_t off_b,
                                         uint32_t vb, bool do_b) {
  if (c.N == 1 || !(do_a || do_b)) return;
#ifndef EMB_RELAXED_PUBLISH
  fence_acq_rel_sys();
#endif
  for (int s = 0; s < c.N; ++s) {
    char* f = reinterpret_cast<char*>(flags_of(c, s));
    if (do_a) st_relaxed_sys(reinterpret_cast<uint32_t*>(f + off_a) + c.r, va);
    if (do_b) st_relaxed_sys(reinterpret_cast<uint32_t*>(f + off_b) + c.r, vb);
  }
}
__device__ __forceinline__ void publish(const DevCtx& c, size_t field_off, uint32_t v) {
  publish2(c, field_off, v, true, 0, 0, false);
}
#define EMB_FLAG_OFF(member) offsetof(::emb::Flags, member)

// ----------------------------------------------------------------- programmatic dependent launch
// Every exchange kernel is launched with the PDL attribute: its grid may start
// while the previous kernel on the stream drains; griddepcontrol.wait (first
// thing in every kernel) blocks until that kernel has completed and its
// memory is visible, and launch_dependents (at the end of every CTA) lets the
// next kernel's launch overlap this one's tail.  Without the attribute both
// are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ----------------------------------------------------------------- vector access
__device__ __forceinline__ uint4 ld16(const void* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ uint4 ld16_nc(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld16_cg(const void* p) { return __ldcg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ void st16(void* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }

// 16 bytes -> floats (EPV = 4 for fp32, 8 for bf16)
template <int DT>
struct Vec;
template <>
struct Vec<F32> {
  static constexpr int EPV = 4;
  __device__ __forceinline__ static void unpack(uint4 u, float* f) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
  __device__ __forceinline__ static uint4 pack(const float* f) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
  }
};
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t bf_pack2(float a, float b) {
  // round-to-nearest-even to bf16 (cvt.rn.bf16x2.f32 d, hi, lo)
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
template <>
struct Vec<BF16> {
  static constexpr int EPV = 8;
  __device__ __forceinline__ static void unpack(uint4 u, float* f) {
    f[0] = bf_lo(u.x); f[1] = bf_hi(u.x); f[2] = bf_lo(u.y); f[3] = bf_hi(u.y);
    f[4] = bf_lo(u.z); f[5] = bf_hi(u.z); f[6] = bf_lo(u.w); f[7] = bf_hi(u.w);
  }
  __device__ __forceinline__ static uint4 pack(const float* f) {
    return make_uint4(bf_pack2(f[0], f[1]), bf_pack2(f[2], f[3]), bf_pack2(f[4], f[5]), bf_pack2(f[6], f[7]));
  }
};

}  // namespace emb
