// k_fwd.cu — forward exchange.
//
// PAPER.md:280 (§4.1.3): "embedding in each process firstly looks up all
// training data of this step and produces a different embedding result.  Then
// AlltoAll is called for redistributing the embedding results so that each
// process gets one embedding result minibatch".  Fig. 3 caption.
//
// B200 design: the lookup + AlltoAll + column concat is
// ONE pull kernel.  Rank r reads, for every token j of its own minibatch and
// every owner s, the 16-byte vectors of shard_s[ids[j], :] straight out of
// s's HBM over NVLink (CUDA IPC mapping) and stores them at their final column
// offset s*d of out[j, :].  One warp per output row (a batch of R rows in
// flight per warp), no staging, no unpack.  The forward needs no id
// all-gather; it still pushes the ids when they were not prefetched, because
// the backward routing of every rank needs every rank's ids (Alg. 1 input
// "gathered training data").
#include <stddef.h>

#include "kernels.cuh"

namespace emb {

static constexpr int FWD_THREADS = 256;
#ifndef EMB_FWD_ROWS
#define EMB_FWD_ROWS 1  // measured (N = 1): 4 -> 1 row per warp, LM 20.5 -> 20.1 us, BERT 45.4 -> 43.3 us
#endif
static constexpr int FWD_ROWS = EMB_FWD_ROWS;  // rows in flight per warp

template <int V>
__global__ void __launch_bounds__(FWD_THREADS) fwd_kernel(DevCtx c, const int* __restrict__ ids, int n,
                                                          char* __restrict__ out, int p, int prefetched,
                                                          int dedup) {
  EMB_TR_ENTRY();
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  const uint32_t t = c.t_rec[p ^ 1] + 1;  // iteration number (device-resident, graph-replay safe)
  EMB_TR_BEGIN(0, t);
  EMB_TR_WAITED(0, t);
  EMB_TR_AT(0, t, 4);
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;
  if (tid == 0) {
    c.t_rec[p] = t;
    if (c.optim == ADAM) {
      // Adam step size of iteration t, once (PyTorch SparseAdam form, readings R3/R4)
      const double td = (double)t;
      c.alpha[p] = (float)((double)c.lr * sqrt(1.0 - pow((double)c.beta2, td)) / (1.0 - pow((double)c.beta1, td)));
    }
    for (int s = 0; s < c.N; ++s) atomicAdd(&c.stats[s], (unsigned long long)n * c.d * c.esz);
    EMB_TR_MID(0, t);
  }
  // (a1) all-gather of this rank's ids into every peer's gids[p][r] (published by route)
  if (!prefetched) {
    for (int i = tid; i < n * c.N; i += nth) {
      const int s = i / n, j = i - s * n;
      gids_of(c, s, p, c.r)[j] = ids[j];
    }
    if (tid < c.N) *ntok_of(c, tid, p, c.r) = n;
    if (tid == 0)
      for (int s = 0; s < c.N; ++s) atomicAdd(&c.stats[2 * c.N + s], (unsigned long long)n * 4ull);
  } else if (c.N > 1) {
    const int* mine = gids_of(c, c.r, p, c.r);  // prefetched by backward(t-1): must be the promised ids
    for (int j = tid; j < n; j += nth)
      if (mine[j] != ids[j]) atomicOr(c.err, ERR_STATE);
    if (tid == 0 && *ntok_of(c, c.r, p, c.r) != n) atomicOr(c.err, ERR_STATE);
  }
  // N == 1 and prefetched: the sort of this batch read next_ids directly (no
  // copy to order against): the ids are fingerprinted here; the gate before
  // the coalesce compares (k_gate.cu GATE_SORTED).  (Fingerprinting after the
  // gather measured mixed in round 1 — LM -0.06 us, BERT +0.3 us — not kept.)
  if (prefetched && c.N == 1) {
    unsigned h = 0;
    for (int j = tid; j < n; j += nth) h += prefetch_hash(__ldg(ids + j), j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0 && h) atomicAdd(&c.fp[p * 4 + 0], h);
    if (tid == 0) atomicAdd(&c.fp[p * 4 + 1], (unsigned)n);
  }
  // every owner applied the prior part of t-1 and the scheduled part of t-2:
  // the gate before this kernel (N > 1) waited for their flags

  // (a2-a4) pull-gather: warp per row; lane holds 16-byte chunks c16 = lane + 32 v
  const int lane = threadIdx.x & 31;
  const int gw = tid >> 5, nw = nth >> 5;
  const size_t slice_bytes = (size_t)c.d * c.esz, row_bytes = (size_t)c.D * c.esz;
  const char* src_base[V];
  int src_off[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int c16 = lane + 32 * v;
    const int s = c16 / c.cps;
    src_base[v] = (c16 < c.cpr) ? shard_of(c, s) : nullptr;
    src_off[v] = (c16 - s * c.cps) * 16;
  }
  // dedup: 1 = N > 1, decided by GATE_FWD (fwd_dd[p]: sort(t) already complete);
  //        2 = N == 1 with the stream joined on sort(t) (always complete)
  if (dedup == 2 || (dedup == 1 && c.fwd_dd[p])) {
    // prefetched, and the sort of this batch is complete: every distinct row is pulled once per reduce chunk (<= C equal
    // ids, ascending positions) and stored to all of the chunk's positions —
    // the NVLink bytes of the forward drop from T_r to ~(U_r + Zipf-head chunks)
    // rows (forward dedup).  Dropped keys (pad when
    // pad_id >= 0, out-of-range ids) sort last and are gathered one by one.
    const size_t bpn = pn(c, p, c.r) * (size_t)c.max_tok;
    const int* cnt = counts_of(c, p, c.r);
    const int NCH = cnt[CNT_NCH], U = cnt[CNT_U];
    const int4* desc = c.chunk_desc + pn(c, p, c.r) * (size_t)c.max_chunks;
    const int* perm = c.perm + bpn;
    const int* uid = c.uid + bpn;
    const int tail0 = c.useg[pn(c, p, c.r) * (size_t)(c.max_tok + 1) + U];
    const int ntail = n - tail0;
    const int items = NCH + (ntail + 31) / 32;
    for (int it = gw; it < items; it += nw) {
      if (it < NCH) {
        const int4 dsc = desc[it];  // {unique, perm begin, perm end, chunks}
        const int id = __ldg(uid + dsc.x);
        const int j = dsc.y + lane;
        const int mypos = (j < dsc.z) ? __ldg(perm + j) : 0;
        uint4 buf[V];
#pragma unroll
        for (int v = 0; v < V; ++v)
          buf[v] = (src_base[v] != nullptr) ? ld16_nc(src_base[v] + (size_t)id * slice_bytes + src_off[v])
                                            : make_uint4(0, 0, 0, 0);
        for (int q = 0; q < dsc.z - dsc.y; ++q) {
          const int pos = __shfl_sync(0xffffffffu, mypos, q);
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const int c16 = lane + 32 * v;
            if (c16 < c.cpr) st16(out + (size_t)pos * row_bytes + (size_t)c16 * 16, buf[v]);
          }
        }
      } else {
        const int j = tail0 + (it - NCH) * 32 + lane;
        const int mypos = (j < n) ? __ldg(perm + j) : -1;
        const int myid = (mypos >= 0) ? __ldg(ids + mypos) : 0;
        for (int q = 0; q < 32; ++q) {
          const int pos = __shfl_sync(0xffffffffu, mypos, q);
          const int id = __shfl_sync(0xffffffffu, myid, q);
          if (pos < 0) break;
          const bool ok = (unsigned)id < (unsigned long long)c.L;
          if (!ok && lane == 0) atomicOr(c.err, ERR_ID);
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const int c16 = lane + 32 * v;
            uint4 x = make_uint4(0, 0, 0, 0);
            if (ok && src_base[v] != nullptr) x = ld16_nc(src_base[v] + (size_t)id * slice_bytes + src_off[v]);
            if (c16 < c.cpr) st16(out + (size_t)pos * row_bytes + (size_t)c16 * 16, x);
          }
        }
      }
    }
  } else
  for (int j0 = gw * FWD_ROWS; j0 < n; j0 += nw * FWD_ROWS) {
    int id[FWD_ROWS];
#pragma unroll
    for (int rr = 0; rr < FWD_ROWS; ++rr) id[rr] = (j0 + rr < n) ? __ldg(ids + j0 + rr) : 0;
    uint4 buf[FWD_ROWS][V];
#pragma unroll
    for (int rr = 0; rr < FWD_ROWS; ++rr) {
      const bool ok = (unsigned)id[rr] < (unsigned long long)c.L;
      if (j0 + rr < n && !ok && lane == 0) atomicOr(c.err, ERR_ID);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        buf[rr][v] = make_uint4(0, 0, 0, 0);
        if (j0 + rr < n && ok && src_base[v] != nullptr)
          buf[rr][v] = ld16_nc(src_base[v] + (size_t)id[rr] * slice_bytes + src_off[v]);
      }
    }
#pragma unroll
    for (int rr = 0; rr < FWD_ROWS; ++rr) {
      if (j0 + rr < n) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int c16 = lane + 32 * v;
          if (c16 < c.cpr) st16(out + (size_t)(j0 + rr) * row_bytes + (size_t)c16 * 16, buf[rr][v]);
        }
      }
    }
  }
  EMB_TR_END(0, t);
  pdl_trigger();
}

// ------------------------------------------------------------------ N == 1: bulk-copy (TMA) gather
// With one process the whole row lives in this GPU's shard, so the gather is a
// row copy W[id] -> Y[j].  fwd_bulk moves rows with the Blackwell bulk-copy
// engine instead of registers: a CTA stages R rows per stage in shared memory
// (cp.async.bulk global -> shared, one 16-byte-multiple row per lane of warp 0,
// completion counted on an mbarrier), then writes them out with
// cp.async.bulk shared -> global; two stages, so the loads of batch i+1 are in
// flight while batch i drains.  Invalid ids get a zero row (generic stores)
// and the sticky ERR_ID, as in fwd_kernel.
#ifndef EMB_FWD_BULK_THREADS
#define EMB_FWD_BULK_THREADS 128
#endif
static constexpr int FB_THREADS = EMB_FWD_BULK_THREADS;
static constexpr int FB_STAGES = 2;

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int NG>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NG) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__global__ void __launch_bounds__(FB_THREADS) fwd_bulk_kernel(DevCtx c, const int* __restrict__ ids, int n,
                                                             char* __restrict__ out, int p, int prefetched, int R) {
  EMB_TR_ENTRY();
  extern __shared__ __align__(128) unsigned char fb_smem[];
  __shared__ __align__(8) uint64_t bars[FB_STAGES];
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  const uint32_t t = c.t_rec[p ^ 1] + 1;
  EMB_TR_BEGIN(0, t);
  EMB_TR_WAITED(0, t);
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;
  if (tid == 0) {  // the forward's per-iteration bookkeeping (as fwd_kernel)
    c.t_rec[p] = t;
    if (c.optim == ADAM) {
      const double td = (double)t;
      c.alpha[p] = (float)((double)c.lr * sqrt(1.0 - pow((double)c.beta2, td)) / (1.0 - pow((double)c.beta1, td)));
    }
    atomicAdd(&c.stats[0], (unsigned long long)n * c.d * c.esz);
  }
  if (!prefetched) {  // (a1) at N == 1: the ids are this rank's own gathered batch
    for (int j = tid; j < n; j += nth) gids_of(c, 0, p, 0)[j] = ids[j];
    if (tid == 0) {
      *ntok_of(c, 0, p, 0) = n;
      atomicAdd(&c.stats[2], (unsigned long long)n * 4ull);
    }
  } else {  // prefetch check: fingerprint of the ids the sort read (k_gate.cu / k_bwd.cu compare)
    unsigned h = 0;
    for (int j = tid; j < n; j += nth) h += prefetch_hash(__ldg(ids + j), j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0 && h) atomicAdd(&c.fp[p * 4 + 0], h);
    if (tid == 0) atomicAdd(&c.fp[p * 4 + 1], (unsigned)n);
  }
  const uint32_t rowB = (uint32_t)c.D * c.esz;
  const char* shard = shard_of(c, 0);
  if (threadIdx.x == 0) {
    for (int st = 0; st < FB_STAGES; ++st) mbar_init(&bars[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int it = 0;
  for (int j0 = blockIdx.x * R; j0 < n; j0 += gridDim.x * R, ++it) {
    const int st = it & (FB_STAGES - 1);
    const uint32_t par = (uint32_t)(it / FB_STAGES) & 1u;
    unsigned char* buf = fb_smem + (size_t)st * R * rowB;
    if (w == 0) {
      // the stage's previous bulk stores (issued FB_STAGES batches ago by this
      // warp) must have finished reading its shared memory
      if (it >= FB_STAGES) bulk_wait_read<FB_STAGES - 1>();
      __syncwarp();
      const int j = j0 + lane;
      const bool valid = lane < R && j < n;
      const int id = valid ? __ldg(ids + j) : 0;
      const bool ok = valid && (unsigned)id < (unsigned long long)c.L;
      const unsigned okm = __ballot_sync(0xffffffffu, ok);
      if (lane == 0) mbar_expect_tx(&bars[st], (uint32_t)__popc(okm) * rowB);
      __syncwarp();
      if (ok) bulk_load(buf + (size_t)lane * rowB, shard + (size_t)id * rowB, rowB, &bars[st]);
      if (valid && !ok) {  // invalid id: zero row, sticky error
        atomicOr(c.err, ERR_ID);
        for (uint32_t o = 0; o < rowB; o += 16) st16(out + (size_t)j * rowB + o, make_uint4(0, 0, 0, 0));
      }
      mbar_wait(&bars[st], par);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (ok) bulk_store(out + (size_t)j * rowB, buf + (size_t)lane * rowB, rowB);
      bulk_commit();
    }
  }
  if (w == 0) bulk_wait_all();  // Y complete before the grid completes (the next kernel reads it)
  EMB_TR_END(0, t);
  pdl_trigger();
}

// rows per stage x CTAs per SM: 4 x 8 measured best for the LM (19.75 vs 19.92 us
// per step with 16 x 3; forward span 4.0 vs 4.5 us — profiles/r02_tune/fwd_bulk.txt)
#ifndef EMB_FWD_BULK_ROWS
#define EMB_FWD_BULK_ROWS 4
#endif
#ifndef EMB_FWD_BULK_PER_SM
#define EMB_FWD_BULK_PER_SM 8
#endif
static int fwd_bulk_rows(const DevCtx& c) {
  int R = EMB_FWD_BULK_ROWS;  // rows per stage (one per lane of warp 0)
  while (R > 1 && (size_t)FB_STAGES * R * c.D * c.esz > 128 * 1024) R >>= 1;
  return R;
}

cudaError_t fwd_bulk_set_smem(const DevCtx& c) {
  const size_t smem = (size_t)FB_STAGES * fwd_bulk_rows(c) * c.D * c.esz;
  return cudaFuncSetAttribute((const void*)fwd_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_fwd(const DevCtx& c, const LaunchCfg& L, const int* ids, int n, void* out, int p,
                       int prefetched, int dedup, cudaStream_t s) {
  if (c.N == 1 && dedup == 0 && L.fwd_bulk) {
    const int R = fwd_bulk_rows(c);
    int grid = (n + R - 1) / R;
    if (grid > L.nsm * EMB_FWD_BULK_PER_SM) grid = L.nsm * EMB_FWD_BULK_PER_SM;
    if (grid < 1) grid = 1;
    const size_t smem = (size_t)FB_STAGES * R * c.D * c.esz;
    return launch_pdl(fwd_bulk_kernel, dim3(grid), dim3(FB_THREADS), smem, s, c, ids, n, static_cast<char*>(out), p,
                      prefetched, R);
  }
  const int warps = (n + FWD_ROWS - 1) / FWD_ROWS;
  int grid = (warps + FWD_THREADS / 32 - 1) / (FWD_THREADS / 32);
  if (grid < 1) grid = 1;
  if (grid > L.nsm * L.fwd_per_sm) grid = L.nsm * L.fwd_per_sm;  // leaves room for other streams
  const int V = (c.cpr + 31) / 32;
  char* o = static_cast<char*>(out);
  const dim3 g(grid), b(FWD_THREADS);
  if (V <= 1) return launch_pdl(fwd_kernel<1>, g, b, 0, s, c, ids, n, o, p, prefetched, dedup);
  if (V <= 2) return launch_pdl(fwd_kernel<2>, g, b, 0, s, c, ids, n, o, p, prefetched, dedup);
  if (V <= 4) return launch_pdl(fwd_kernel<4>, g, b, 0, s, c, ids, n, o, p, prefetched, dedup);
  if (V <= 8) return launch_pdl(fwd_kernel<8>, g, b, 0, s, c, ids, n, o, p, prefetched, dedup);
  return cudaErrorInvalidValue;
}

cudaError_t preload_fwd() {
  for (const void* f : {(const void*)fwd_kernel<1>, (const void*)fwd_kernel<2>, (const void*)fwd_kernel<4>,
                        (const void*)fwd_kernel<8>, (const void*)fwd_bulk_kernel})
    if (cudaError_t e = preload(f)) return e;
  return cudaSuccess;
}

}  // namespace emb
