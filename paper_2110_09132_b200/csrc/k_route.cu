// k_route.cu — per-source sort / unique (a6) and the Alg. 1 split + routing
// tables (a5, a8) of SURVEY §8(a).
//
// Alg. 1, lines 2-5:
//   G_coalesced <- COALESCE(G)        — rows of equal id are summed (values: by
//                                       k_bwd.cu; here: the segments of equal ids,
//                                       PAPER.md:349-352)
//   D_u <- UNIQUE(D_cur[n])           — ascending unique ids of source n
//   i_prior <- D_u ∩ D_next           — D_next = gathered next batch (reading R1),
//   i_scheduled <- D_u \ i_prior        "always keep the data of the next
//                                       iteration in memory"
// "The calculations require a considerable computing resource, and the GPU
// idle time after BP is a good occasion".
//
// B200 design.  The expensive part — sorting every source's (id, position)
// pairs — depends only on the gathered ids of iteration t, which the prefetch
// makes available one iteration early.  So it is split off:
//
//   sort_kernel(t)   one CTA (1024 threads) per source, on an auxiliary stream,
//                    launched as soon as ids(t) are gathered (normally right
//                    after route(t-1)); it overlaps coal/merge of t-1 and the
//                    forward of t.  LSD radix sort in shared memory over the
//                    drop+id bits (stable => positions ascending inside a
//                    segment); 4-bit digits ranked with thread-private u16
//                    counters and one raking block scan per pass.  Output:
//                    perm (positions in (dropped, id, pos) order), the ascending
//                    unique kept ids uid[] and their segment starts useg[].
//   route_kernel(t)  on the main stream in the backward ("after BP"): pushes
//                    the next ids (prefetch all-gather), builds D_next as an
//                    L-bit shared-memory bitmap, splits the unique ids into
//                    prior / scheduled with a stable ballot partition (slot k:
//                    prior ascending, then scheduled ascending), and emits the
//                    slot tables, reduce chunks (C rows) and the multi-chunk
//                    (Zipf-head) slot list.  Every rank does every source (the
//                    owner merge needs all of them), so no size messages are
//                    exchanged (reading R14).
#include <stddef.h>

#include "kernels.cuh"

namespace emb {

static constexpr int RT_THREADS = 1024;
static constexpr int RT_WARPS = RT_THREADS / 32;
static constexpr int DBITS = 4;          // digit bits per radix pass
static constexpr int NDIG = 1 << DBITS;  // 16 digits
static constexpr int RAKE = NDIG;        // u16 counters scanned per thread

// Block-wide exclusive scan of one int per thread; *total receives the sum.
__device__ __forceinline__ int block_exscan(int v, int* tmp, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = (lane < RT_WARPS) ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    tmp[lane] = s;
  }
  __syncthreads();
  const int before = (w > 0) ? tmp[w - 1] : 0;
  *total = tmp[RT_WARPS - 1];
  __syncthreads();
  return before + x - v;
}

// Two-counter exclusive scan of per-warp totals held in wa[32], wb[32] by
// warp 0; results back in place, grand totals in tot[0..1].
__device__ __forceinline__ void warp_totals_scan(int* wa, int* wb, int* tot) {
  const int lane = threadIdx.x & 31;
  if ((threadIdx.x >> 5) == 0) {
    const int x = wa[lane], y = wb[lane];
    int sx = x, sy = y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, sx, o), b = __shfl_up_sync(0xffffffffu, sy, o);
      if (lane >= o) { sx += a; sy += b; }
    }
    wa[lane] = sx - x;
    wb[lane] = sy - y;
    if (lane == 31) { tot[0] = sx; tot[1] = sy; }
  }
  __syncthreads();
}

// ============================================================== sort (aux stream)
template <typename K, int EPT>
__global__ void __launch_bounds__(RT_THREADS, 1) sort_kernel(DevCtx c, int p, int fwd_pushed) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int kb = (c.max_tok + 1 + 3) & ~3;  // keys per buffer, 16-byte aligned
  K* keyA = reinterpret_cast<K*>(smem_raw);
  K* keyB = keyA + kb;
  uint16_t* cnt = reinterpret_cast<uint16_t*>(keyB + kb);  // [NDIG][RT_THREADS]
  int* tmp = reinterpret_cast<int*>(cnt + NDIG * RT_THREADS);
  __shared__ int s_tot[2];

  const int n = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  // t of the batch being sorted: this kernel runs either after forward(t) (ids
  // pushed there) or after route(t-1) (prefetched) — before forward(t) wrote
  // t_rec[p] — so derive it from the previous iteration's record.
  const uint32_t tt = c.t_rec[p ^ 1] + 1;
  EMB_TS(20);
  if (n == 0 && tid == 0 && fwd_pushed) publish(c, EMB_FLAG_OFF(ids), tt);
  if (tid == 0 && c.N > 1) wait_flag(c, &flags_of(c, c.r)->ids[n], tt);
  __syncthreads();

  const int T = __ldcg(ntok_of(c, c.r, p, n));
  const int* g = gids_of(c, c.r, p, n);
  const int posbits = c.posbits, idbits = c.idbits;
  const int dshift = posbits + idbits;
  const long long L = c.L;
  {
    int cur[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int i = tid + k * RT_THREADS;
      cur[k] = (i < T) ? __ldcg(g + i) : 0;
    }
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int i = tid + k * RT_THREADS;
      if (i < T) {
        int id = cur[k];
        int drop = 0;
        if ((unsigned)id >= (unsigned long long)L) {
          id = (int)L;  // invalid: sentinel, dropped
          drop = 1;
        } else if (c.pad_id >= 0 && (long long)id == c.pad_id) {
          drop = 1;
        }
        keyA[i] = (K(drop) << dshift) | (K(id) << posbits) | K(i);
      }
    }
  }
  __syncthreads();
  EMB_TS(21);

  // LSD radix passes over [posbits, dshift + 1): blocked keys, private counters
  const int b0 = tid * EPT;
  const int topbit = dshift + 1;
  for (int shift = posbits; shift < topbit; shift += DBITS) {
    const unsigned dmask = (1u << min(DBITS, topbit - shift)) - 1u;
    K kk[EPT];
    int dg[EPT], rk[EPT];
#pragma unroll
    for (int d = 0; d < NDIG; ++d) cnt[d * RT_THREADS + tid] = 0;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      if (b0 + e < T) {
        kk[e] = keyA[b0 + e];
        dg[e] = (int)((unsigned)(kk[e] >> shift) & dmask);
        uint16_t* cp = &cnt[dg[e] * RT_THREADS + tid];
        rk[e] = *cp;
        *cp = (uint16_t)(rk[e] + 1);
      }
    }
    __syncthreads();
    {  // raking exclusive scan over (digit-major, thread-minor) counters
      uint4* rp = reinterpret_cast<uint4*>(cnt + tid * RAKE);
      const uint4 a = rp[0], b = rp[1];
      uint32_t wv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      int loc[RAKE];
      int sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        loc[2 * q] = (int)(wv[q] & 0xFFFFu);
        loc[2 * q + 1] = (int)(wv[q] >> 16);
      }
#pragma unroll
      for (int q = 0; q < RAKE; ++q) {
        const int x = loc[q];
        loc[q] = sum;
        sum += x;
      }
      int tot;
      const int ex = block_exscan(sum, tmp, &tot);
#pragma unroll
      for (int q = 0; q < 8; ++q) wv[q] = (uint32_t)(loc[2 * q] + ex) | ((uint32_t)(loc[2 * q + 1] + ex) << 16);
      rp[0] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      rp[1] = make_uint4(wv[4], wv[5], wv[6], wv[7]);
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < EPT; ++e)
      if (b0 + e < T) keyB[cnt[dg[e] * RT_THREADS + tid] + rk[e]] = kk[e];
    __syncthreads();
    K* sw = keyA; keyA = keyB; keyB = sw;
  }
  EMB_TS(22);

  // heads -> unique kept ids (ascending) + segment starts; perm = sorted positions
  const size_t bpn = pn(c, p, n) * (size_t)c.max_tok;
  int* perm = c.perm + bpn;
  int* uid = c.uid + bpn;
  int* useg = c.useg + pn(c, p, n) * (size_t)(c.max_tok + 1);
  const K posmask = (K(1) << posbits) - 1;
  const unsigned idmask = (1u << idbits) - 1u;
  const int per_warp = (T + RT_WARPS - 1) / RT_WARPS;
  const int w0 = min(T, w * per_warp), w1 = min(T, w0 + per_warp);
  int* wa = tmp;
  int* wb = tmp + 32;
  {
    int kept = 0;
    for (int base = w0; base < w1; base += 32) {
      const int i = base + lane;
      const bool valid = i < w1;
      const K key = valid ? keyA[i] : K(0);
      const bool head = valid && (i == 0 || (key >> posbits) != (keyA[i - 1] >> posbits));
      kept += __popc(__ballot_sync(0xffffffffu, head && (key >> dshift) == 0));
    }
    if (lane == 0) { wa[w] = kept; wb[w] = 0; }
    __syncthreads();
    warp_totals_scan(wa, wb, s_tot);
  }
  int kbase = wa[w];
  const int U = s_tot[0];
  __syncthreads();
  for (int base = w0; base < w1; base += 32) {
    const int i = base + lane;
    const bool valid = i < w1;
    const K key = valid ? keyA[i] : K(0);
    const K prev = (valid && i > 0) ? keyA[i - 1] : K(0);
    const bool head = valid && (i == 0 || (key >> posbits) != (prev >> posbits));
    const bool kept = head && (key >> dshift) == 0;
    const unsigned keptm = __ballot_sync(0xffffffffu, kept);
    if (valid) {
      perm[i] = (int)(key & posmask);
      if (kept) {
        const int k = kbase + __popc(keptm & lt_mask);
        uid[k] = (int)((key >> posbits) & idmask);
        useg[k] = i;
      } else if (head && (i == 0 || (prev >> dshift) == 0)) {
        useg[U] = i;  // first dropped element = end of the last kept segment
      }
    }
    kbase += __popc(keptm);
  }
  if (tid == 0) {
    // end of the last kept segment when nothing is dropped (a dropped head wrote it otherwise)
    int* cn = c.counts + pn(c, p, n) * CNT_W;
    cn[CNT_ST] = T;
    cn[CNT_SU] = U;
  }
  __syncthreads();
  if (tid == 0 && (T == 0 || (keyA[T - 1] >> dshift) == 0)) useg[U] = T;
  EMB_TS(23);
  pdl_trigger();
}

// ============================================================== route (main stream)
template <int EPT>
__global__ void __launch_bounds__(RT_THREADS, 1) route_kernel(DevCtx c, int p, const int* __restrict__ next_ids,
                                                              int n_next) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem_raw);  // D_next, ceil(L/32) words
  __shared__ int s_tmp[64];
  __shared__ int s_tot[2];

  const int n = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint32_t t = c.t_rec[p];
  const int p1 = p ^ 1;
  const bool split = (c.mode == SPLIT);
  const bool has_next = (next_ids != nullptr);
  const long long L = c.L;
  EMB_TS(0);
  if (n == 0 && tid == 0 && c.optim == ADAM) {
    // Adam step size of this iteration, once (PyTorch SparseAdam form, reading R3/R4)
    const double td = (double)t;
    c.alpha[p] = (float)((double)c.lr * sqrt(1.0 - pow((double)c.beta2, td)) / (1.0 - pow((double)c.beta1, td)));
  }

  // ---- 1. prefetch all-gather: CTA n pushes this rank's next ids to peer n
  if (has_next) {
    int* dst = gids_of(c, n, p1, c.r);
    int v[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int j = tid + k * RT_THREADS;
      if (j < n_next) v[k] = __ldg(next_ids + j);
    }
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int j = tid + k * RT_THREADS;
      if (j < n_next) dst[j] = v[k];
    }
    if (tid == 0) {
      *ntok_of(c, n, p1, c.r) = n_next;
      atomicAdd(&c.stats[2 * c.N + n], (unsigned long long)n_next * 4ull);
    }
    __syncthreads();
    if (tid == 0 && c.N > 1) {
      __threadfence_system();
      st_release_sys(&flags_of(c, n)->ids[c.r], t + 1);
    }
  }

  // ---- 2. unique ids of source n (from sort(t)) into registers
  const int* cn = counts_of(c, p, n);
  const int U = cn[CNT_SU];
  const int Tn = cn[CNT_ST];
  const size_t bpn = pn(c, p, n) * (size_t)c.max_tok;
  const int* uid = c.uid + bpn;
  const int* useg = c.useg + pn(c, p, n) * (size_t)(c.max_tok + 1);
  // warp-contiguous ranges of unique ids, lane-striped rounds
  const int per_w = (U + RT_WARPS - 1) / RT_WARPS;
  const int k0w = min(U, w * per_w), k1w = min(U, k0w + per_w);
  constexpr int RMAX = (EPT * RT_THREADS / RT_WARPS + 31) / 32;  // rounds per warp (U <= max_tok)
  int uv[RMAX], sa[RMAX], sb[RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    const int k = k0w + r * 32 + lane;
    uv[r] = (k < k1w) ? uid[k] : -1;
    sa[r] = (k < k1w) ? useg[k] : 0;
    sb[r] = (k < k1w) ? useg[k + 1] : 0;
  }
  EMB_TS(1);

  // ---- 3. D_next bitmap (gathered next batch of every rank)
  if (split && has_next) {
    const int nwords = (int)((L + 31) >> 5);
    for (int i = tid; i < nwords; i += RT_THREADS) bitmap[i] = 0u;
    if (tid == 0) wait_all(c, flags_of(c, c.r)->ids, t + 1);
    __syncthreads();
    for (int s = 0; s < c.N; ++s) {
      const int cnx = __ldcg(ntok_of(c, c.r, p1, s));
      const int* gn = gids_of(c, c.r, p1, s);
      int v[EPT];
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const int j = tid + k * RT_THREADS;
        v[k] = (j < cnx) ? __ldcg(gn + j) : -1;
      }
#pragma unroll
      for (int k = 0; k < EPT; ++k)
        if ((unsigned)v[k] < (unsigned long long)L) atomicOr(&bitmap[v[k] >> 5], 1u << (v[k] & 31));
    }
    __syncthreads();
  }
  EMB_TS(2);

  // ---- 4. stable partition of the unique ids: prior (in D_next) first
  auto is_prior = [&](int id) {
    return !split || (has_next && ((bitmap[id >> 5] >> (id & 31)) & 1u));
  };
  int* wa = s_tmp;
  int* wb = s_tmp + 32;
  {
    int pri = 0, nch_sum = 0;
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      const bool valid = uv[r] >= 0;
      pri += __popc(__ballot_sync(0xffffffffu, valid && is_prior(uv[r])));
    }
    if (lane == 0) { wa[w] = pri; wb[w] = nch_sum; }
    __syncthreads();
    warp_totals_scan(wa, wb, s_tot);
  }
  const int P_tot = s_tot[0];
  int pbase = wa[w];                 // prior heads before this warp
  int dbase = k0w - wa[w];           // scheduled heads before this warp (k0w = all heads before)
  __syncthreads();
  int* slot_id = c.slot_id + bpn;
  int* seg_start = c.seg_start + bpn;
  int* seg_end = c.seg_end + bpn;
  int kslot[RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    const bool valid = uv[r] >= 0;
    const bool pr = valid && is_prior(uv[r]);
    const unsigned pm = __ballot_sync(0xffffffffu, pr);
    const unsigned dm = __ballot_sync(0xffffffffu, valid && !pr);
    kslot[r] = -1;
    if (valid) {
      const int k = pr ? pbase + __popc(pm & lt_mask) : P_tot + dbase + __popc(dm & lt_mask);
      kslot[r] = k;
      slot_id[k] = uv[r];
      seg_start[k] = sa[r];
      seg_end[k] = sb[r];
      if (c.N > 1) c.slotmap[(size_t)uv[r] * c.N + n] = ((unsigned long long)t << 32) | (unsigned)k;
    }
    pbase += __popc(pm);
    dbase += __popc(dm);
  }
  __syncthreads();  // slot tables complete (block scope)
  EMB_TS(3);

  // ---- 5. reduce chunks in slot order (C rows each) and the long-slot list
  int* chunk_off = c.chunk_off + pn(c, p, n) * (size_t)(c.max_tok + 1);
  int* chunk_slot = c.chunk_slot + pn(c, p, n) * (size_t)c.max_chunks;
  int* long_slots = c.long_slots + pn(c, p, n) * (size_t)c.max_long;
  int nch[RMAX], kk[RMAX];
  {
    int wch = 0, wlg = 0;
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      const int k = k0w + r * 32 + lane;  // slot-ordered walk (global memory, block-visible)
      kk[r] = k;
      int x = (k < k1w) ? (seg_end[k] - seg_start[k] + c.C - 1) / c.C : 0;
      nch[r] = x;
      wlg += __popc(__ballot_sync(0xffffffffu, x > 1));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      wch += x;
    }
    if (lane == 0) { wa[w] = wch; wb[w] = wlg; }
    __syncthreads();
    warp_totals_scan(wa, wb, s_tot);
  }
  const int NCH = s_tot[0], NLONG = s_tot[1];
  {
    int cb = wa[w], lb = wb[w];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      const int k = kk[r];
      const bool valid = k < k1w;
      int incl = nch[r];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned longm = __ballot_sync(0xffffffffu, nch[r] > 1);
      if (valid) {
        const int off = cb + incl - nch[r];
        chunk_off[k] = off;
        for (int q = 0; q < nch[r]; ++q) chunk_slot[off + q] = k;
        if (nch[r] > 1) long_slots[lb + __popc(longm & lt_mask)] = k;
      }
      cb += __shfl_sync(0xffffffffu, incl, 31);
      lb += __popc(longm);
    }
  }
  if (tid == 0) {
    chunk_off[U] = NCH;
    int* cw = c.counts + pn(c, p, n) * CNT_W;
    cw[CNT_T] = Tn;
    cw[CNT_U] = U;
    cw[CNT_P] = P_tot;
    cw[CNT_NCH] = NCH;
    cw[CNT_NLONG] = NLONG;
  }
  (void)kslot;
  EMB_TS(4);
  pdl_trigger();
}

// ============================================================== launchers
static int ept_for(int max_tok) {
  const int need = (max_tok + RT_THREADS - 1) / RT_THREADS;
  const int opts[] = {1, 2, 4, 5, 8, 12, 16};
  for (int e : opts)
    if (e >= need) return e;
  return -1;
}

size_t sort_smem_bytes(int max_tok, bool key64) {
  return (size_t)2 * ((max_tok + 1 + 3) & ~3) * (key64 ? 8 : 4) + (size_t)NDIG * RT_THREADS * 2 + 64 * 4;
}

size_t route_smem_bytes(long long vocab) { return (size_t)((vocab + 31) / 32) * 4 + 16; }

template <typename K>
static void* sort_fn(int ept) {
  switch (ept) {
    case 1: return (void*)sort_kernel<K, 1>;
    case 2: return (void*)sort_kernel<K, 2>;
    case 4: return (void*)sort_kernel<K, 4>;
    case 5: return (void*)sort_kernel<K, 5>;
    case 8: return (void*)sort_kernel<K, 8>;
    case 12: return (void*)sort_kernel<K, 12>;
    case 16: return (void*)sort_kernel<K, 16>;
  }
  return nullptr;
}

static void* route_fn(int ept) {
  switch (ept) {
    case 1: return (void*)route_kernel<1>;
    case 2: return (void*)route_kernel<2>;
    case 4: return (void*)route_kernel<4>;
    case 5: return (void*)route_kernel<5>;
    case 8: return (void*)route_kernel<8>;
    case 12: return (void*)route_kernel<12>;
    case 16: return (void*)route_kernel<16>;
  }
  return nullptr;
}

cudaError_t route_set_smem(int max_tok, bool key64, size_t sort_smem, size_t route_smem) {
  const int e = ept_for(max_tok);
  void* f = key64 ? sort_fn<unsigned long long>(e) : sort_fn<uint32_t>(e);
  void* g = route_fn(e);
  if (!f || !g) return cudaErrorInvalidValue;
  cudaError_t st = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sort_smem);
  if (st != cudaSuccess) return st;
  return cudaFuncSetAttribute(g, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)route_smem);
}

cudaError_t launch_sort(const DevCtx& c, int p, int fwd_pushed, bool key64, size_t smem, cudaStream_t s) {
  void* f = key64 ? sort_fn<unsigned long long>(ept_for(c.max_tok)) : sort_fn<uint32_t>(ept_for(c.max_tok));
  if (!f) return cudaErrorInvalidValue;
  DevCtx cc = c;
  void* args[] = {&cc, &p, &fwd_pushed};
  return launch_pdl_raw(f, dim3(c.N), dim3(RT_THREADS), smem, s, args);
}

cudaError_t launch_route(const DevCtx& c, int p, const int* next_ids, int n_next, size_t smem, cudaStream_t s) {
  void* f = route_fn(ept_for(c.max_tok));
  if (!f) return cudaErrorInvalidValue;
  DevCtx cc = c;
  void* args[] = {&cc, &p, &next_ids, &n_next};
  return launch_pdl_raw(f, dim3(c.N), dim3(RT_THREADS), smem, s, args);
}

}  // namespace emb
