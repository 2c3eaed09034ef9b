// k_route.cu — per-source sort / unique / reduce chunks (a6), the prefetch
// all-gather + D_next marks (a5) and the Alg. 1 slot tables (a8) of SURVEY §8(a).
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
// B200 design:
//   sort_kernel(t)   one CTA (1024 threads) per source on an auxiliary stream,
//                    launched as soon as ids(t) are gathered — normally right
//                    after mark(t-1), one iteration ahead — so it overlaps the
//                    previous backward and the forward.  LSD radix sort in
//                    shared memory over the drop+id bits (stable => positions
//                    ascending inside a segment), 4-bit digits ranked with
//                    thread-private u16 counters and one raking block scan per
//                    pass.  Emits perm, the ascending unique kept ids uid[i],
//                    their segments useg[i], the reduce chunks (C rows) per
//                    unique, the multi-chunk (Zipf-head) list and, N > 1, the
//                    owner routing slotmap[id][n] = (t, i).
//   mark_kernel(t)   main stream: CTA n pushes this rank's next ids to peer n
//                    (the prefetch all-gather) and, in SPLIT, marks D_next:
//                    nextmark[p][id] = t+1 (epoch tag, never cleared).  The
//                    split is then a per-id test in every backward kernel — no
//                    prefix over the split on the critical path.
//   tables_kernel(t) off the critical path: the Alg. 1 split in the paper's
//                    presentation — slot k = prior ids ascending, then
//                    scheduled ids ascending (P_n ++ D_n) and p_n — for the
//                    statistics and the integer parity tests.
//   Every rank sorts every source (the owner merge needs all of them; the
//   gathered ids are local), so no size messages are exchanged (reading R14).
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

// Two-counter exclusive scan of per-warp totals wa[32], wb[32] (warp 0 does
// it); results back in place, grand totals in tot[0..1].
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
__global__ void __launch_bounds__(RT_THREADS, 1) sort_kernel(DevCtx c, int p, const int* own_ids, int own_n) {
  EMB_TR_ENTRY();
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int kb = (c.max_tok + 1 + 3) & ~3;  // keys per buffer (+1 for segs[U]), 16-byte aligned
  K* keyA = reinterpret_cast<K*>(smem_raw);
  K* keyB = keyA + kb;
  uint16_t* cnt = reinterpret_cast<uint16_t*>(keyB + kb);  // [NDIG][RT_THREADS]
  int* tmp = reinterpret_cast<int*>(cnt + NDIG * RT_THREADS);
  __shared__ int s_tot[2];

  const int n = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  // t of the batch being sorted: this kernel runs either after forward(t) (ids
  // pushed there) or after mark(t-1) (prefetched) — possibly before forward(t)
  // wrote t_rec[p] — so derive it from the previous iteration's record.
  const uint32_t tt = c.t_rec[p ^ 1] + 1;
  EMB_TR_BEGIN(1, tt);
  // N > 1: the gate before this kernel published / waited the ids flags.
  // own_ids (N == 1 prefetch): this rank's batch is read straight from the caller.

  const bool own = own_ids != nullptr && n == c.r;
  const int T = own ? own_n : __ldcg(ntok_of(c, c.r, p, n));
  const int* g = own ? own_ids : gids_of(c, c.r, p, n);
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
          id = (int)L;  // invalid: sentinel, dropped (the forward flags EMB_ERR_ID_RANGE)
          drop = 1;
        } else if (c.pad_id >= 0 && (long long)id == c.pad_id) {
          drop = 1;     // reading R6: pad rows get no gradient
        }
        keyA[i] = (K(drop) << dshift) | (K(id) << posbits) | K(i);
      }
    }
  }
  __syncthreads();

  EMB_TR_AT(1, tt, 4);
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

  EMB_TR_AT(1, tt, 5);
  // ---- heads -> unique kept ids (ascending), segments, owner routing
  const size_t bpn = pn(c, p, n) * (size_t)c.max_tok;
  int* perm = c.perm + bpn;
  int* uid = c.uid + bpn;
  int* useg = c.useg + pn(c, p, n) * (size_t)(c.max_tok + 1);
  int* segs = reinterpret_cast<int*>(keyB);  // shared copy of useg (keyB is free)
  const K posmask = (K(1) << posbits) - 1;
  const unsigned idmask = (1u << idbits) - 1u;
  int* wa = tmp;
  int* wb = tmp + 32;
  const int per_warp = (T + RT_WARPS - 1) / RT_WARPS;
  const int w0 = min(T, w * per_warp), w1 = min(T, w0 + per_warp);
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
  if (tid == 0) segs[U] = T;  // end of the last kept segment (a dropped head overwrites it)
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
        const int id = (int)((key >> posbits) & idmask);
        uid[k] = id;
        segs[k] = i;
        if (c.N > 1)
          c.slotmap[((size_t)p * c.L + id) * c.N + n] = ((unsigned long long)tt << 32) | (unsigned)k;
      } else if (head && (i == 0 || (prev >> dshift) == 0)) {
        segs[U] = i;  // first dropped element = end of the last kept segment
      }
    }
    kbase += __popc(keptm);
  }
  __syncthreads();

  EMB_TR_AT(1, tt, 6);
  // ---- reduce chunks (C rows) per unique, chunk -> unique, multi-chunk list
  int* chunk_off = c.chunk_off + pn(c, p, n) * (size_t)(c.max_tok + 1);
  int4* chunk_desc = c.chunk_desc + pn(c, p, n) * (size_t)c.max_chunks;
  int* long_u = c.long_u + pn(c, p, n) * (size_t)c.max_long;
  const int per_w = (U + RT_WARPS - 1) / RT_WARPS;
  const int k0w = min(U, w * per_w), k1w = min(U, k0w + per_w);
  {
    int wch = 0, wlg = 0;
    for (int base = k0w; base < k1w; base += 32) {
      const int k = base + lane;
      int x = (k < k1w) ? (segs[k + 1] - segs[k] + c.C - 1) / c.C : 0;
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
    for (int base = k0w; base < k1w; base += 32) {
      const int k = base + lane;
      const bool valid = k < k1w;
      const int a = valid ? segs[k] : 0, b = valid ? segs[k + 1] : 0;
      const int nch = valid ? (b - a + c.C - 1) / c.C : 0;
      int incl = nch;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned longm = __ballot_sync(0xffffffffu, nch > 1);
      if (valid) {
        const int off = cb + incl - nch;
        useg[k] = a;
        chunk_off[k] = off;
        for (int q = 0; q < nch; ++q) chunk_desc[off + q] = make_int4(k, a + q * c.C, min(b, a + (q + 1) * c.C), nch);
        if (nch > 1) long_u[lb + __popc(longm & lt_mask)] = k;
      }
      cb += __shfl_sync(0xffffffffu, incl, 31);
      lb += __popc(longm);
    }
  }
  if (tid == 0) {
    useg[U] = segs[U];
    chunk_off[U] = NCH;
    int* cn = c.counts + pn(c, p, n) * CNT_W;
    cn[CNT_T] = T;
    cn[CNT_U] = U;
    cn[CNT_NCH] = NCH;
    cn[CNT_NLONG] = NLONG;
  }
  EMB_TR_END(1, tt);
  pdl_trigger();
}

// ============================================================== mark (main stream)
// CTA s pushes this rank's next ids to peer s (prefetch all-gather; the flag is
// released by that CTA after its own stores), then with do_mark (SPLIT) all
// CTAs wait for every rank's next ids and tag D_next: nextmark[p][id] = t+1.
__global__ void __launch_bounds__(1024) mark_kernel(DevCtx c, int p, const int* __restrict__ next_ids, int n_next,
                                                    int do_mark) {
  EMB_TR_ENTRY();
  pdl_wait();
  const uint32_t t = c.t_rec[p];
  EMB_TR_BEGIN(2, t);
  const int p1 = p ^ 1;
  const int tid = threadIdx.x;
  constexpr int MK = 16;  // ids per thread in flight: max_tok <= 16 * 1024
  if (next_ids != nullptr) {
    int v[MK];
#pragma unroll
    for (int k = 0; k < MK; ++k) {
      const int j = tid + k * 1024;
      v[k] = (j < n_next) ? __ldg(next_ids + j) : 0;
    }
    for (int s = blockIdx.x; s < c.N; s += gridDim.x) {
      int* dst = gids_of(c, s, p1, c.r);
#pragma unroll
      for (int k = 0; k < MK; ++k) {
        const int j = tid + k * 1024;
        if (j < n_next) dst[j] = v[k];
      }
      if (tid == 0) {
        *ntok_of(c, s, p1, c.r) = n_next;
        atomicAdd(&c.stats[2 * c.N + s], (unsigned long long)n_next * 4ull);
      }
      __syncthreads();
      EMB_TR_AT(2, t, 4);
      if (tid == 0 && c.N > 1) {
        fence_acq_rel_sys();  // cumulative over the CTA's stores (ordered by the barrier)
        EMB_TR_AT(2, t, 5);
        st_relaxed_sys(&flags_of(c, s)->ids[c.r], t + 1);
      }
    }
  }
  EMB_TR_MID(2, t);
  if (do_mark && next_ids != nullptr) {
    if (tid == 0) wait_all(c, flags_of(c, c.r)->ids, t + 1);  // grid = N CTAs: co-resident
    __syncthreads();
    EMB_TR_WAITED(2, t);
    int* mark = c.nextmark + (size_t)p * c.L;
    const int nthr = gridDim.x * blockDim.x, gtid = blockIdx.x * blockDim.x + tid;
    for (int s = 0; s < c.N; ++s) {
      const int cn = __ldcg(ntok_of(c, c.r, p1, s));
      const int* gn = gids_of(c, c.r, p1, s);
      for (int j0 = gtid; j0 < cn; j0 += MK * nthr) {
        int id[MK];
#pragma unroll
        for (int k = 0; k < MK; ++k) {
          const int j = j0 + k * nthr;
          id[k] = (j < cn) ? __ldcg(gn + j) : -1;
        }
#pragma unroll
        for (int k = 0; k < MK; ++k)
          if ((unsigned)id[k] < (unsigned long long)c.L) mark[id[k]] = (int)(t + 1);
      }
    }
  }
  EMB_TR_END(2, t);
  pdl_trigger();
}

// ============================================================== Alg. 1 tables (off the critical path)
// Slot order of the paper's presentation: P_n = U_n ∩ D_next ascending, then
// D_n = U_n \ P_n ascending (a stable ballot partition of the unique ids).
template <int EPT>
__global__ void __launch_bounds__(RT_THREADS, 1) tables_kernel(DevCtx c, int p) {
  EMB_TR_ENTRY();
  pdl_wait();
  __shared__ int s_tmp[64];
  __shared__ int s_tot[2];
  const int n = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint32_t t = c.t_rec[p];
  EMB_TR_BEGIN(9, t);
  const int U = counts_of(c, p, n)[CNT_U];
  const size_t bpn = pn(c, p, n) * (size_t)c.max_tok;
  const int* uid = c.uid + bpn;
  int* slot_id = c.slot_id + bpn;
  const int per_w = (U + RT_WARPS - 1) / RT_WARPS;
  const int k0w = min(U, w * per_w), k1w = min(U, k0w + per_w);
  constexpr int RMAX = EPT;  // rounds per warp: U <= max_tok <= EPT * 1024
  int uv[RMAX];
  bool pr[RMAX];
  int pri = 0;
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    const int k = k0w + r * 32 + lane;
    uv[r] = (k < k1w) ? uid[k] : -1;
  }
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    pr[r] = uv[r] >= 0 && is_prior(c, p, t, uv[r]);
    pri += __popc(__ballot_sync(0xffffffffu, pr[r]));
  }
  if (lane == 0) { s_tmp[w] = pri; s_tmp[32 + w] = 0; }
  __syncthreads();
  warp_totals_scan(s_tmp, s_tmp + 32, s_tot);
  const int P_tot = s_tot[0];
  int pbase = s_tmp[w];
  int dbase = k0w - s_tmp[w];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    const bool valid = uv[r] >= 0;
    const unsigned pm = __ballot_sync(0xffffffffu, pr[r]);
    const unsigned dm = __ballot_sync(0xffffffffu, valid && !pr[r]);
    if (valid) slot_id[pr[r] ? pbase + __popc(pm & lt_mask) : P_tot + dbase + __popc(dm & lt_mask)] = uv[r];
    pbase += __popc(pm);
    dbase += __popc(dm);
  }
  if (tid == 0) c.counts[pn(c, p, n) * CNT_W + CNT_P] = P_tot;
  EMB_TR_END(9, t);
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

static void* tables_fn(int ept) {
  switch (ept) {
    case 1: return (void*)tables_kernel<1>;
    case 2: return (void*)tables_kernel<2>;
    case 4: return (void*)tables_kernel<4>;
    case 5: return (void*)tables_kernel<5>;
    case 8: return (void*)tables_kernel<8>;
    case 12: return (void*)tables_kernel<12>;
    case 16: return (void*)tables_kernel<16>;
  }
  return nullptr;
}

cudaError_t sort_set_smem(int max_tok, bool key64, size_t smem) {
  void* f = key64 ? sort_fn<unsigned long long>(ept_for(max_tok)) : sort_fn<uint32_t>(ept_for(max_tok));
  if (!f) return cudaErrorInvalidValue;
  return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_sort(const DevCtx& c, int p, const int* own_ids, int own_n, bool key64, size_t smem,
                        cudaStream_t s) {
  void* f = key64 ? sort_fn<unsigned long long>(ept_for(c.max_tok)) : sort_fn<uint32_t>(ept_for(c.max_tok));
  if (!f) return cudaErrorInvalidValue;
  DevCtx cc = c;
  void* args[] = {&cc, &p, &own_ids, &own_n};
  return launch_pdl_raw(f, dim3(c.N), dim3(RT_THREADS), smem, s, args);
}

cudaError_t launch_mark(const DevCtx& c, const LaunchCfg& L, int p, const int* next_ids, int n_next, int do_mark,
                        cudaStream_t s) {
  (void)L;
  return launch_pdl(mark_kernel, dim3(c.N), dim3(1024), 0, s, c, p, next_ids, n_next, do_mark);
}

cudaError_t launch_tables(const DevCtx& c, int p, cudaStream_t s) {
  void* f = tables_fn(ept_for(c.max_tok));
  if (!f) return cudaErrorInvalidValue;
  DevCtx cc = c;
  void* args[] = {&cc, &p};
  return launch_pdl_raw(f, dim3(c.N), dim3(RT_THREADS), 0, s, args);
}

}  // namespace emb
