// k_route.cu — per-source sort / unique / Alg. 1 split / routing tables
// (SURVEY §8(a) a6 + a8).
//
// Alg. 1, lines 2-5:
//   G_coalesced <- COALESCE(G)        — rows of equal id summed (the values are
//                                       summed later by k_bwd.cu; here: the
//                                       segments of equal ids)
//   D_u <- UNIQUE(D_cur[n])           — ascending unique ids of source n
//   i_prior <- D_u ∩ D_next           — nextmark[id] == t+1 (reading R1: D_next
//   i_scheduled <- D_u \ i_prior        is the gathered next batch)
// "The calculations require a considerable computing resource, and the GPU
// idle time after BP is a good occasion".
//
// B200 design: one CTA (1024 threads) per source n; every rank computes every
// source (the owner merge needs all of them, and the gathered ids are already
// local), so no size messages are exchanged (reading R14).  Keys
// (id << posbits | pos) live in shared memory and are sorted by an LSD radix
// sort over the id bits only (stable => positions stay ascending inside a
// segment).  Each pass ranks digits with __match_any_sync warp multisplit,
// one (digit, warp) counter table and one block scan.  Outputs (global):
//   perm[i]      positions in (id, pos) order
//   slot k       prior slots 0..p-1 (ascending id), then scheduled p..u-1
//   slot_id[k], seg_start[k], seg_end[k]   segment of slot k inside perm
//   chunk_off[k] first reduce chunk of slot k (C rows per chunk), chunk_slot[]
//   slotmap[id][n] = (t << 32) | k         (epoch-tagged, never cleared)
//   counts = {T, u, p, nchunks}
#include "kernels.cuh"

namespace emb {

static constexpr int RT_THREADS = 1024;
static constexpr int RT_WARPS = RT_THREADS / 32;
static constexpr int RADIX_BITS = 8;
static constexpr int RADIX = 1 << RADIX_BITS;

// Block-wide exclusive scan of one int per thread; returns the exclusive
// prefix and writes the total to *total.  `tmp` >= 33 ints of shared memory.
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
    tmp[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  const int before = (w > 0) ? tmp[w - 1] : 0;
  *total = tmp[RT_WARPS - 1];
  __syncthreads();
  return before + x - v;
}

template <typename K>
__device__ __forceinline__ int key_id(K k, int posbits) { return (int)(k >> posbits); }

template <typename K>
__global__ void __launch_bounds__(RT_THREADS, 1) route_kernel(DevCtx c, int p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* keyA = reinterpret_cast<K*>(smem_raw);
  K* keyB = keyA + c.max_tok;
  int* hist = reinterpret_cast<int*>(keyB + c.max_tok);  // [RADIX][RT_WARPS]
  int* tmp = hist + RADIX * RT_WARPS;                     // scan scratch (64 ints)

  const int n = blockIdx.x;  // source rank
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t t = c.t_rec[p];
  if (tid == 0) wait_flag(c, &flags_of(c, c.r)->ids[n], t);
  __syncthreads();

  const int T = __ldcg(ntok_of(c, c.r, p, n));
  const int* g = gids_of(c, c.r, p, n);
  const int posbits = c.posbits;
  const K posmask = (K(1) << posbits) - 1;
  const long long L = c.L;

  // load (id, pos) keys; invalid ids map to the sentinel L (sorted last, dropped)
  for (int i = tid; i < T; i += RT_THREADS) {
    int id = __ldcg(g + i);
    if ((unsigned)id >= (unsigned long long)L) id = (int)L;
    keyA[i] = (K(id) << posbits) | K(i);
  }
  __syncthreads();

  // ---- LSD radix sort over the id bits (stable) --------------------------------
  const int per_warp = (T + RT_WARPS - 1) / RT_WARPS;
  const int w0 = min(T, w * per_warp), w1 = min(T, w0 + per_warp);
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int shift = posbits; shift < posbits + c.idbits; shift += RADIX_BITS) {
    const int nb = min(RADIX_BITS, posbits + c.idbits - shift);
    const unsigned dmask = (1u << nb) - 1u;
    for (int i = tid; i < RADIX * RT_WARPS; i += RT_THREADS) hist[i] = 0;
    __syncthreads();
    // count: hist[digit][warp]
    for (int base = w0; base < w1; base += 32) {
      const int i = base + lane;
      const bool valid = i < w1;
      const unsigned am = __ballot_sync(0xffffffffu, valid);
      if (valid) {
        const unsigned dg = (unsigned)(keyA[i] >> shift) & dmask;
        const unsigned peers = __match_any_sync(am, dg);
        if (lane == __ffs(peers) - 1) hist[dg * RT_WARPS + w] += __popc(peers);
      }
      __syncwarp();
    }
    __syncthreads();
    // exclusive scan over (digit-major, warp-minor): 8 entries per thread
    {
      int loc[RADIX * RT_WARPS / RT_THREADS];
      int sum = 0;
#pragma unroll
      for (int k = 0; k < RADIX * RT_WARPS / RT_THREADS; ++k) {
        loc[k] = hist[tid * (RADIX * RT_WARPS / RT_THREADS) + k];
        sum += loc[k];
      }
      int tot;
      int ex = block_exscan(sum, tmp, &tot);
#pragma unroll
      for (int k = 0; k < RADIX * RT_WARPS / RT_THREADS; ++k) {
        hist[tid * (RADIX * RT_WARPS / RT_THREADS) + k] = ex;
        ex += loc[k];
      }
    }
    __syncthreads();
    // scatter (stable: warp ranges in order, rounds in order, lanes in order)
    for (int base = w0; base < w1; base += 32) {
      const int i = base + lane;
      const bool valid = i < w1;
      const unsigned am = __ballot_sync(0xffffffffu, valid);
      unsigned peers = 0, dg = 0;
      int b = 0;
      K k = 0;
      if (valid) {
        k = keyA[i];
        dg = (unsigned)(k >> shift) & dmask;
        peers = __match_any_sync(am, dg);
        b = hist[dg * RT_WARPS + w];
        keyB[b + __popc(peers & lt_mask)] = k;
      }
      __syncwarp();
      if (valid && lane == __ffs(peers) - 1) hist[dg * RT_WARPS + w] = b + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    K* sw = keyA; keyA = keyB; keyB = sw;
  }

  // ---- segments, Alg. 1 split, slot numbering ----------------------------------
  // per-head packed counter: bits 0-14 prior heads, 15-29 scheduled heads,
  // 30-31 dropped heads (pad / invalid sentinel)
  const size_t base_pn = pn(c, p, n) * (size_t)c.max_tok;
  const int ept = (T + RT_THREADS - 1) / RT_THREADS;
  const int i0 = min(T, tid * ept), i1 = min(T, i0 + ept);
  const bool split = (c.mode == SPLIT);
  auto dropped = [&](int id) { return id >= L || (c.pad_id >= 0 && (long long)id == c.pad_id); };
  auto is_prior = [&](int id) { return !split || c.nextmark[id] == (int)(t + 1); };
  int local = 0;
  for (int i = i0; i < i1; ++i) {
    const int id = key_id(keyA[i], posbits);
    const bool head = (i == 0) || id != key_id(keyA[i - 1], posbits);
    if (head) local += dropped(id) ? (1 << 30) : (is_prior(id) ? 1 : (1 << 15));
  }
  int total;
  int run = block_exscan(local, tmp, &total);
  const int P_tot = total & 0x7FFF, Q_tot = (total >> 15) & 0x7FFF, U_tot = P_tot + Q_tot;

  int* perm = c.perm + base_pn;
  int* slot_id = c.slot_id + base_pn;
  int* seg_start = c.seg_start + base_pn;
  int* seg_end = c.seg_end + base_pn;
  unsigned long long* slotmap = c.slotmap;
  bool cur_prior = false;
  for (int i = i0; i < i1; ++i) {
    const K key = keyA[i];
    const int id = key_id(key, posbits);
    const bool head = (i == 0) || id != key_id(keyA[i - 1], posbits);
    const bool tail = (i == T - 1) || id != key_id(keyA[i + 1], posbits);
    perm[i] = (int)(key & posmask);
    if (dropped(id)) {
      if (head) run += 1 << 30;
      continue;
    }
    if (head) {
      cur_prior = is_prior(id);
      run += cur_prior ? 1 : (1 << 15);
    } else if (i == i0) {
      cur_prior = is_prior(id);  // segment began in another thread's range
    }
    const int k = cur_prior ? (run & 0x7FFF) - 1 : P_tot + ((run >> 15) & 0x7FFF) - 1;
    if (head) {
      slot_id[k] = id;
      seg_start[k] = i;
      slotmap[(size_t)id * c.N + n] = ((unsigned long long)t << 32) | (unsigned)k;
    }
    if (tail) seg_end[k] = i + 1;
  }
  __syncthreads();

  // ---- reduce chunks: C rows per chunk, prefix over slots -----------------------
  int* chunk_off = c.chunk_off + pn(c, p, n) * (size_t)(c.max_tok + 1);
  int* chunk_slot = c.chunk_slot + pn(c, p, n) * (size_t)c.max_chunks;
  const int ept2 = (U_tot + RT_THREADS - 1) / RT_THREADS;
  const int k0 = min(U_tot, tid * ept2), k1 = min(U_tot, k0 + ept2);
  int lc = 0;
  for (int k = k0; k < k1; ++k) lc += (seg_end[k] - seg_start[k] + c.C - 1) / c.C;
  int ctot;
  int cex = block_exscan(lc, tmp, &ctot);
  for (int k = k0; k < k1; ++k) {
    const int nch = (seg_end[k] - seg_start[k] + c.C - 1) / c.C;
    chunk_off[k] = cex;
    for (int q = 0; q < nch; ++q) chunk_slot[cex + q] = k;
    cex += nch;
  }
  if (tid == 0) {
    chunk_off[U_tot] = ctot;
    int* cnt = c.counts + pn(c, p, n) * 4;
    cnt[0] = T;
    cnt[1] = U_tot;
    cnt[2] = P_tot;
    cnt[3] = ctot;
  }
}

size_t route_smem_bytes(int max_tok, bool key64) {
  return (size_t)2 * max_tok * (key64 ? 8 : 4) + (size_t)RADIX * RT_WARPS * 4 + 64 * 4;
}

cudaError_t route_set_smem(bool key64, size_t smem) {
  if (key64)
    return cudaFuncSetAttribute(route_kernel<unsigned long long>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return cudaFuncSetAttribute(route_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_route(const DevCtx& c, const LaunchCfg& L, int p, bool key64, size_t smem, cudaStream_t s) {
  (void)L;
  if (key64)
    route_kernel<unsigned long long><<<c.N, RT_THREADS, smem, s>>>(c, p);
  else
    route_kernel<uint32_t><<<c.N, RT_THREADS, smem, s>>>(c, p);
  return cudaGetLastError();
}

}  // namespace emb
