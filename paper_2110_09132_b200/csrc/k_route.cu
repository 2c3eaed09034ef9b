// k_route.cu — the prefetch all-gather + D_next marks (a5) and the Alg. 1
// slot tables (a8) of SURVEY §8(a).  (The per-source sort / unique / reduce
// chunks of a6 are in k_sort.cu.)
//
// Alg. 1, lines 2-5:
//   D_u <- UNIQUE(D_cur[n])           — ascending unique ids of source n (k_sort.cu)
//   i_prior <- D_u ∩ D_next           — D_next = gathered next batch (reading R1),
//   i_scheduled <- D_u \ i_prior        "always keep the data of the next
//                                       iteration in memory"
//
// B200 design:
//   markpush(t)      pushes this rank's next ids to every peer (the prefetch
//                    all-gather); the following gate publishes them
//   marktag(t)       in SPLIT, marks D_next: nextmark[p][id] = t+1 (epoch tag,
//                    never cleared).  The split is then a per-id test in every
//                    backward kernel — no prefix over the split on the
//                    critical path.
//   tables_kernel(t) off the critical path: the Alg. 1 split in the paper's
//                    presentation — slot k = prior ids ascending, then
//                    scheduled ids ascending (P_n ++ D_n) and p_n — for the
//                    statistics and the integer parity tests.
#include <stddef.h>

#include "kernels.cuh"

namespace emb {

static constexpr int RT_THREADS = 1024;
static constexpr int RT_WARPS = RT_THREADS / 32;

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

// ============================================================== mark (a5)
// markpush: CTA (s, k) stores slice k of this rank's next ids into peer s's
// gids[p^1][r] (the prefetch all-gather).  No flag and no fence here: the gate
// that follows on the stream publishes ids(t+1) after this grid completed.
static constexpr int MP_SLICES = 4;   // CTAs per destination
static constexpr int MP_THREADS = 256;
static constexpr int MK = 8;          // ids in flight per thread
__global__ void __launch_bounds__(MP_THREADS) markpush_kernel(DevCtx c, int p, const int* __restrict__ next_ids,
                                                             int n_next, int t_mode) {
  EMB_TR_ENTRY();
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  // t of this batch: N > 1 the sort of t precedes on this stream (DESIGN B7);
  // N == 1 (side stream) the side stream's own count of backward calls
  if (t_mode && blockIdx.x == 0 && threadIdx.x == 0) c.side_it[0] += 1;
  const uint32_t t = t_mode ? c.side_it[0] + 1 : __ldcg(c.sorted + p);
  (void)t;
  EMB_TR_BEGIN(2, t);
  EMB_TR_WAITED(2, t);
  const int s = blockIdx.x % c.N, k = blockIdx.x / c.N;
  int* dst = gids_of(c, s, p ^ 1, c.r);
  const int stride = MP_SLICES * MP_THREADS;
  for (int j0 = k * MP_THREADS + threadIdx.x; j0 < n_next; j0 += MK * stride) {
    int v[MK];
#pragma unroll
    for (int q = 0; q < MK; ++q) {
      const int j = j0 + q * stride;
      v[q] = (j < n_next) ? __ldg(next_ids + j) : 0;
    }
#pragma unroll
    for (int q = 0; q < MK; ++q) {
      const int j = j0 + q * stride;
      if (j < n_next) dst[j] = v[q];
    }
  }
  // next_ids == NULL (N == 1 only: the side stream's iteration counter above
  // still advances): no copy and no count — forward(t+1) writes its own count
  // on the main stream, which a late store of 0 here would overwrite
  if (next_ids != nullptr && k == 0 && threadIdx.x == 0) {
    *ntok_of(c, s, p ^ 1, c.r) = n_next;
    atomicAdd(&c.stats[2 * c.N + s], (unsigned long long)n_next * 4ull);
  }
  EMB_TR_END(2, t);
  pdl_trigger();
}

// marktag: with every rank's next ids here (N > 1: the gate before waited the
// ids flags), tag D_next: nextmark[p][id] = t+1 (epoch tag, never cleared), so
// the split is a per-id test everywhere.  Then the completion flag marked[p].
static constexpr int MT_CTAS_PER_SRC = 8;
__global__ void __launch_bounds__(MP_THREADS) marktag_kernel(DevCtx c, int p, int do_mark, int set_flag, int t_mode) {
  EMB_TR_ENTRY();
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  const uint32_t t = t_mode ? __ldcg(c.side_it) : __ldcg(c.sorted + p);  // see markpush
  EMB_TR_BEGIN(17, t);
  EMB_TR_WAITED(17, t);
  if (blockIdx.x == 0 && threadIdx.x < 2) c.plan_cnt[p * 2 + threadIdx.x] = 0;  // re-arm the plan of parity p
  if (do_mark) {
    int* mark = c.nextmark + (size_t)p * c.L;
    const int nthr = gridDim.x * blockDim.x, gtid = blockIdx.x * blockDim.x + threadIdx.x;
    for (int s = 0; s < c.N; ++s) {
      const int cn = __ldcg(ntok_of(c, c.r, p ^ 1, s));
      const int* gn = gids_of(c, c.r, p ^ 1, s);
      for (int j0 = gtid; j0 < cn; j0 += MK * nthr) {
        int id[MK];
#pragma unroll
        for (int q = 0; q < MK; ++q) {
          const int j = j0 + q * nthr;
          id[q] = (j < cn) ? __ldcg(gn + j) : -1;
        }
#pragma unroll
        for (int q = 0; q < MK; ++q)
          if ((unsigned)id[q] < (unsigned long long)c.L) mark[id[q]] = (int)(t + 1);
      }
    }
  }
  // completion flag for the gates of the main stream (the apply, the next
  // forward); N > 1 the plan kernel that follows sets it instead
  __syncthreads();
  if (set_flag && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&c.mark_cnt[p], 1u) == gridDim.x - 1) {
      c.mark_cnt[p] = 0;
      __threadfence();
      st_release_gpu(&c.marked[p], t);
    }
  }
  EMB_TR_END(17, t);
  pdl_trigger();
}

// ============================================================== owner merge plan (N > 1)
// Thread per (source n, unique i): the lowest source holding the id (slotmap
// tag == t) emits one plan entry {id, i at every source or -1} into the part
// of the id (SPLIT: prior iff in D_next).  The merge kernels then walk their
// part's entries: no slotmap / D_next lookups and no idle items on the
// critical path, and the scheduled merge no longer reads the routing tables
// (so the sort of t+1 only waits for this rank's scheduled push of t-1).
__global__ void __launch_bounds__(MP_THREADS) plan_kernel(DevCtx c, int p) {
  EMB_TR_ENTRY();
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  const uint32_t t = __ldcg(c.sorted + p);  // t of this batch: sort(t) precedes on this stream (DESIGN B7)
  EMB_TR_BEGIN(19, t);
  EMB_TR_WAITED(19, t);
  int cnt[EMB_WMAX];
  int total = 0;
#pragma unroll
  for (int n = 0; n < EMB_WMAX; ++n) {
    cnt[n] = (n < c.N) ? counts_of(c, p, n)[CNT_U] : 0;
    total += cnt[n];
  }
  const int PW = 1 + c.N;
  for (int item = blockIdx.x * blockDim.x + threadIdx.x; item < total; item += gridDim.x * blockDim.x) {
    int n = 0, k = item;
#pragma unroll
    for (int m = 0; m < EMB_WMAX - 1; ++m)
      if (n == m && k >= cnt[m]) { k -= cnt[m]; n = m + 1; }
    const int u = c.uid[pn(c, p, n) * (size_t)c.max_tok + k];
    const unsigned long long* sm = c.slotmap + ((size_t)p * c.L + u) * c.N;
    int ks[EMB_WMAX];
    bool leader = true;
#pragma unroll
    for (int n2 = 0; n2 < EMB_WMAX; ++n2) {
      ks[n2] = -1;
      if (n2 < c.N) {
        const unsigned long long e = (n2 == n) ? (((unsigned long long)t << 32) | (unsigned)k) : sm[n2];
        if ((uint32_t)(e >> 32) == t) {
          ks[n2] = (int)(uint32_t)e;
          if (n2 < n) leader = false;
        }
      }
    }
    const int part = (c.mode == SPLIT && !is_prior(c, p, t, u)) ? 1 : 0;
    // warp-aggregated slot allocation: one atomic per (warp, part), not per entry
    // (the order of plan entries is free: every entry is one id's whole merge)
    const unsigned act = __activemask();
    const unsigned m1 = __ballot_sync(act, leader && part == 1), m0 = __ballot_sync(act, leader && part == 0);
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int base0 = 0, base1 = 0;
    const int first = __ffs(act) - 1;
    if (lane == first) {
      if (m0) base0 = atomicAdd(&c.plan_cnt[p * 2 + 0], __popc(m0));
      if (m1) base1 = atomicAdd(&c.plan_cnt[p * 2 + 1], __popc(m1));
    }
    base0 = __shfl_sync(act, base0, first);
    base1 = __shfl_sync(act, base1, first);
    if (!leader) continue;
    const int slot = part ? base1 + __popc(m1 & lt) : base0 + __popc(m0 & lt);
    int* e = c.plan + (((size_t)p * 2 + part) * c.N * c.max_tok + slot) * PW;
    e[0] = u;
#pragma unroll
    for (int n2 = 0; n2 < EMB_WMAX; ++n2)
      if (n2 < c.N) e[1 + n2] = ks[n2];
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // completion flag (marked[p]: D_next tags and plan are complete)
    __threadfence();
    if (atomicAdd(&c.mark_cnt[p], 1u) == gridDim.x - 1) {
      c.mark_cnt[p] = 0;
      __threadfence();
      st_release_gpu(&c.marked[p], t);
    }
  }
  EMB_TR_END(19, t);
  pdl_trigger();
}

// ============================================================== Alg. 1 tables (off the critical path)
// Slot order of the paper's presentation: P_n = U_n ∩ D_next ascending, then
// D_n = U_n \ P_n ascending (a stable ballot partition of the unique ids).
template <int EPT>
__global__ void __launch_bounds__(RT_THREADS, 1) tables_kernel(DevCtx c, int p, int t_mode) {
  EMB_TR_ENTRY();
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  __shared__ int s_tmp[64];
  __shared__ int s_tot[2];
  const int n = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint32_t t = t_mode ? __ldcg(c.side_it) : __ldcg(c.sorted + p);  // see markpush
  EMB_TR_BEGIN(9, t);
  EMB_TR_WAITED(9, t);
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
  const int opts[] = {1, 2, 4, 5, 8, 12, 16, 32};  // 32: up to 32768 uniques (the 16-CTA sort's cap)
  for (int e : opts)
    if (e >= need) return e;
  return -1;
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
    case 32: return (void*)tables_kernel<32>;
  }
  return nullptr;
}

cudaError_t launch_markpush(const DevCtx& c, int p, const int* next_ids, int n_next, int t_mode, cudaStream_t s) {
  return launch_pdl(markpush_kernel, dim3(c.N * MP_SLICES), dim3(MP_THREADS), 0, s, c, p, next_ids, n_next, t_mode);
}

cudaError_t launch_marktag(const DevCtx& c, int p, int do_mark, int set_flag, int t_mode, cudaStream_t s) {
  return launch_pdl(marktag_kernel, dim3(c.N * MT_CTAS_PER_SRC), dim3(MP_THREADS), 0, s, c, p, do_mark, set_flag,
                    t_mode);
}

cudaError_t launch_plan(const DevCtx& c, int p, cudaStream_t s) {
  long long items = (long long)c.N * c.max_tok;
  int grid = (int)((items + MP_THREADS - 1) / MP_THREADS);
  if (grid > 148 * 4) grid = 148 * 4;
  return launch_pdl(plan_kernel, dim3(grid), dim3(MP_THREADS), 0, s, c, p);
}

cudaError_t launch_tables(const DevCtx& c, int p, int t_mode, cudaStream_t s) {
  void* f = tables_fn(ept_for(c.max_tok));
  if (!f) return cudaErrorInvalidValue;
  DevCtx cc = c;
  void* args[] = {&cc, &p, &t_mode};
  return launch_pdl_raw(f, dim3(c.N), dim3(RT_THREADS), 0, s, args);
}

cudaError_t preload_route() {
  for (const void* f : {(const void*)markpush_kernel, (const void*)marktag_kernel, (const void*)plan_kernel,
                        (const void*)tables_kernel<1>, (const void*)tables_kernel<2>,
                        (const void*)tables_kernel<4>, (const void*)tables_kernel<5>, (const void*)tables_kernel<8>,
                        (const void*)tables_kernel<12>, (const void*)tables_kernel<16>,
                        (const void*)tables_kernel<32>})
    if (cudaError_t e = preload(f)) return e;
  return cudaSuccess;
}

}  // namespace emb
