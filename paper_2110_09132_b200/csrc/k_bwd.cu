// k_bwd.cu — backward exchange kernels.
//
// PAPER.md:280 (§4.1.3): "each process computes sparse gradients of embedding
// tables [...] AlltoAll is called again to exchange sparse gradients between
// processes [...] and each process could update all parameters".
// Alg. 1: COALESCE then INDEX_SELECT into the prior part
// (exchanged first, "must be finished before embedding FP") and
// the scheduled part ("delayed", assigned "the latest" priority).
// Modified Adam: one step value t for both parts (reading R3).
//
// B200 design:
//   coal_kernel    sender-side segmented reduce of dY in fp32 (one warp per
//                  chunk of <= C rows, fixed-order two-level combine for long
//                  Zipf-head segments, no float atomics), rounded to the wire
//                  dtype and stored DIRECTLY into each owner's receive rows
//                  over NVLink (prior slots) or into a local stage (scheduled
//                  slots) — COALESCE + INDEX_SELECT + AlltoAll in one pass.
//   defpush_kernel pushes the staged scheduled rows (side stream, later).
//   rawpush/rawcoal RAW mode: raw dY slices travel, the owner coalesces.
//   merge_kernel   owner: sum each row's contributions in ascending source rank
//                  (fp32), scale, fused SGD / Adam update of shard, m, v.
#include "kernels.cuh"

namespace emb {

static constexpr int BWD_THREADS = 256;

// ------------------------------------------------------------------ helpers
template <bool PEER>
__device__ __forceinline__ uint4 ldrow16(const char* p) {
  if (PEER) return __ldcg(reinterpret_cast<const uint4*>(p));  // peer-written rows: read at L2
  return ld16_nc(p);
}

// acc[v*EPV + i] = sum over rows perm[b..e) (ascending) of row[c16 = lane + 32 v]
template <int DT, int V, bool PEER>
__device__ __forceinline__ void reduce_rows(const char* __restrict__ base, size_t stride, int ncol16,
                                            const int* __restrict__ perm, int b, int e, float* acc) {
  constexpr int EPV = Vec<DT>::EPV;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < V * EPV; ++i) acc[i] = 0.f;
  for (int i = b; i < e; i += 4) {
    uint4 buf[4][V];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      if (i + rr < e) {
        const char* row = base + (size_t)__ldg(perm + i + rr) * stride;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int c16 = lane + 32 * v;
          if (c16 < ncol16) buf[rr][v] = ldrow16<PEER>(row + (size_t)c16 * 16);
        }
      }
    }
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      if (i + rr < e) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int c16 = lane + 32 * v;
          if (c16 < ncol16) {
            float f[EPV];
            Vec<DT>::unpack(buf[rr][v], f);
#pragma unroll
            for (int k = 0; k < EPV; ++k) acc[v * EPV + k] += f[k];
          }
        }
      }
    }
  }
}

// Two-level combine of a slot split into nch > 1 chunks.  Every chunk's warp
// stores its partial; the last warp to arrive sums partials 0..nch-1 in chunk
// order (deterministic).  Returns true in the warp that must emit the row.
template <int NA>
__device__ __forceinline__ bool combine_partials(float* __restrict__ part_base /* chunk 0 of this slot */,
                                                 int dw, int chunk_in_slot, int nch, int* ctr, int ncol16,
                                                 int EPV, float* acc) {
  const int lane = threadIdx.x & 31;
  float* mine = part_base + (size_t)chunk_in_slot * dw;
#pragma unroll
  for (int v = 0; v < NA; ++v) {
    const int c16 = lane + 32 * (v / EPV) ;
    if (c16 < ncol16) mine[c16 * EPV + (v % EPV)] = acc[v];
  }
  __threadfence();
  __syncwarp();
  int prev = 0;
  if (lane == 0) prev = atomicAdd(ctr, 1);
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (prev != nch - 1) return false;
  __threadfence();
  if (lane == 0) *ctr = 0;  // re-arm (stream-ordered reuse)
#pragma unroll
  for (int v = 0; v < NA; ++v) acc[v] = 0.f;
  for (int q = 0; q < nch; ++q) {
    const float* pq = part_base + (size_t)q * dw;
#pragma unroll
    for (int v = 0; v < NA; ++v) {
      const int c16 = lane + 32 * (v / EPV);
      if (c16 < ncol16) acc[v] += __ldcg(pq + c16 * EPV + (v % EPV));
    }
  }
  return true;
}

// ------------------------------------------------------------------ sender coalesce
template <int DT, int V>
__global__ void __launch_bounds__(BWD_THREADS) coal_kernel(DevCtx c, const char* __restrict__ dY, int p) {
  constexpr int EPV = Vec<DT>::EPV;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t t = c.t_rec[p];
  const int r = c.r;
  const int* cnt = c.counts + pn(c, p, r) * 4;
  const int Pr = cnt[2], NCH = cnt[3];
  const size_t bpn = pn(c, p, r) * (size_t)c.max_tok;
  const int* perm = c.perm + bpn;
  const int* seg_start = c.seg_start + bpn;
  const int* seg_end = c.seg_end + bpn;
  const int* chunk_off = c.chunk_off + pn(c, p, r) * (size_t)(c.max_tok + 1);
  const int* chunk_slot = c.chunk_slot + pn(c, p, r) * (size_t)c.max_chunks;
  const size_t row_bytes = (size_t)c.D * c.esz;
  const size_t slice_bytes = (size_t)c.d * c.esz;
  float acc[V * EPV];
  for (int ch = gw; ch < NCH; ch += nw) {
    const int k = chunk_slot[ch];
    const int c0 = chunk_off[k], nch = chunk_off[k + 1] - c0;
    const int b = seg_start[k] + (ch - c0) * c.C;
    const int e = min(seg_end[k], b + c.C);
    reduce_rows<DT, V, false>(dY, row_bytes, c.cpr, perm, b, e, acc);
    if (nch > 1) {
      float* part0 = c.scratch + ((size_t)p * c.max_chunks + c0) * c.D;
      if (!combine_partials<V * EPV>(part0, c.D, ch - c0, nch, c.slot_ctr + bpn + k, c.cpr, EPV, acc)) continue;
    }
    // emit: prior slot -> owner s's receive row k (NVLink store); scheduled -> local stage
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int c16 = lane + 32 * v;
      if (c16 < c.cpr) {
        const uint4 val = Vec<DT>::pack(acc + v * EPV);
        if (k < Pr) {
          const int s = c16 / c.cps, cs = c16 - s * c.cps;
          st16(recv_of(c, s, p, r) + (size_t)k * slice_bytes + (size_t)cs * 16, val);
        } else {
          st16(c.stage + ((size_t)p * c.max_tok + (k - Pr)) * row_bytes + (size_t)c16 * 16, val);
        }
      }
    }
  }
  if (last_block_done(&c.done_ctr[K_COAL])) {
    for (int s = 0; s < c.N; ++s) {
      st_release_sys(&flags_of(c, s)->pub[0][r], t);
      atomicAdd(&c.stats[c.N + s], (unsigned long long)Pr * slice_bytes);
    }
  }
}

// ------------------------------------------------------------------ scheduled push
__global__ void __launch_bounds__(BWD_THREADS) defpush_kernel(DevCtx c, int p) {
  const uint32_t t = c.t_rec[p];
  const int r = c.r;
  const int* cnt = c.counts + pn(c, p, r) * 4;
  const int U = cnt[1], Pr = cnt[2], Q = U - Pr;
  const size_t row_bytes = (size_t)c.D * c.esz, slice_bytes = (size_t)c.d * c.esz;
  const size_t total = (size_t)Q * c.cpr;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (size_t q = tid; q < total; q += nth) {
    const int k = (int)(q / c.cpr), c16 = (int)(q - (size_t)k * c.cpr);
    const uint4 val = ld16_nc(c.stage + ((size_t)p * c.max_tok + k) * row_bytes + (size_t)c16 * 16);
    const int s = c16 / c.cps, cs = c16 - s * c.cps;
    st16(recv_of(c, s, p, r) + (size_t)(Pr + k) * slice_bytes + (size_t)cs * 16, val);
  }
  if (last_block_done(&c.done_ctr[K_DEFPUSH])) {
    for (int s = 0; s < c.N; ++s) {
      st_release_sys(&flags_of(c, s)->pub[1][r], t);
      atomicAdd(&c.stats[c.N + s], (unsigned long long)Q * slice_bytes);
    }
  }
}

// ------------------------------------------------------------------ RAW mode
__global__ void __launch_bounds__(BWD_THREADS) rawpush_kernel(DevCtx c, const char* __restrict__ dY, int n, int p) {
  const uint32_t t = c.t_rec[p];
  const int r = c.r;
  const size_t row_bytes = (size_t)c.D * c.esz, slice_bytes = (size_t)c.d * c.esz;
  const size_t total = (size_t)n * c.cpr;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (size_t q = tid; q < total; q += nth) {
    const int j = (int)(q / c.cpr), c16 = (int)(q - (size_t)j * c.cpr);
    const uint4 val = ld16_nc(dY + (size_t)j * row_bytes + (size_t)c16 * 16);
    const int s = c16 / c.cps, cs = c16 - s * c.cps;
    st16(recv_of(c, s, p, r) + (size_t)j * slice_bytes + (size_t)cs * 16, val);
  }
  if (last_block_done(&c.done_ctr[K_RAWPUSH])) {
    for (int s = 0; s < c.N; ++s) {
      st_release_sys(&flags_of(c, s)->pub[0][r], t);
      atomicAdd(&c.stats[c.N + s], (unsigned long long)n * slice_bytes);
    }
  }
}

// owner-side coalesce of every source's raw slices -> gc_owner (fp32)
template <int DT, int V>
__global__ void __launch_bounds__(BWD_THREADS) rawcoal_kernel(DevCtx c, int p) {
  constexpr int EPV = Vec<DT>::EPV;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t t = c.t_rec[p];
  block_wait_all(c, flags_of(c, c.r)->pub[0], t);
  int nchs[EMB_WMAX];
  int total = 0;
#pragma unroll
  for (int n = 0; n < EMB_WMAX; ++n) {
    nchs[n] = (n < c.N) ? c.counts[pn(c, p, n) * 4 + 3] : 0;
    total += nchs[n];
  }
  const size_t slice_bytes = (size_t)c.d * c.esz;
  float acc[V * EPV];
  for (int gch = gw; gch < total; gch += nw) {
    int n = 0, ch = gch;
    while (ch >= nchs[n]) { ch -= nchs[n]; ++n; }
    const size_t bpn = pn(c, p, n) * (size_t)c.max_tok;
    const int* chunk_off = c.chunk_off + pn(c, p, n) * (size_t)(c.max_tok + 1);
    const int k = c.chunk_slot[pn(c, p, n) * (size_t)c.max_chunks + ch];
    const int c0 = chunk_off[k], nch = chunk_off[k + 1] - c0;
    const int b = c.seg_start[bpn + k] + (ch - c0) * c.C;
    const int e = min(c.seg_end[bpn + k], b + c.C);
    reduce_rows<DT, V, true>(recv_of(c, c.r, p, n), slice_bytes, c.cps, c.perm + bpn, b, e, acc);
    if (nch > 1) {
      float* part0 = c.scratch + (size_t)p * c.max_chunks * c.D + ((size_t)n * c.max_chunks + c0) * c.d;
      if (!combine_partials<V * EPV>(part0, c.d, ch - c0, nch, c.slot_ctr + bpn + k, c.cps, EPV, acc)) continue;
    }
    float* dst = c.gc_owner + (bpn + k) * (size_t)c.d;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int c16 = lane + 32 * v;
      if (c16 < c.cps) {
#pragma unroll
        for (int q = 0; q < EPV; q += 4)
          *reinterpret_cast<float4*>(dst + c16 * EPV + q) =
              make_float4(acc[v * EPV + q], acc[v * EPV + q + 1], acc[v * EPV + q + 2], acc[v * EPV + q + 3]);
      }
    }
  }
}

// ------------------------------------------------------------------ owner merge + update
template <int DT, bool RAWSRC>
__global__ void __launch_bounds__(BWD_THREADS) merge_kernel(DevCtx c, int p, int part, int G) {
  constexpr int EPV = Vec<DT>::EPV;
  const uint32_t t = c.t_rec[p];
  if (c.mode != RAW) block_wait_all(c, flags_of(c, c.r)->pub[part], t);
  int lo[EMB_WMAX], cnt[EMB_WMAX];
  int total = 0;
#pragma unroll
  for (int n = 0; n < EMB_WMAX; ++n) {
    lo[n] = cnt[n] = 0;
    if (n < c.N) {
      const int* cn = c.counts + pn(c, p, n) * 4;
      const int U = cn[1], Pr = cn[2];
      lo[n] = part ? Pr : 0;
      cnt[n] = (part ? U : Pr) - lo[n];
      total += cnt[n];
    }
  }
  float alpha = 0.f;
  if (c.optim == ADAM) {
    const double td = (double)t;
    alpha = (float)((double)c.lr * sqrt(1.0 - pow((double)c.beta2, td)) / (1.0 - pow((double)c.beta1, td)));
  }
  const float om_b1 = 1.f - c.beta1, om_b2 = 1.f - c.beta2;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int grp = gtid / G, gl = gtid - grp * G, ngrp = (gridDim.x * blockDim.x) / G;
  const size_t slice_bytes = (size_t)c.d * c.esz;
  char* shard = shard_of(c, c.r);
  for (int item = grp; item < total; item += ngrp) {
    int n = 0, rem = item;
    while (rem >= cnt[n]) { rem -= cnt[n]; ++n; }
    const int k = lo[n] + rem;
    const int u = c.slot_id[pn(c, p, n) * (size_t)c.max_tok + k];
    const unsigned long long* sm = c.slotmap + (size_t)u * c.N;
    unsigned long long ent[EMB_WMAX];
    bool leader = true;
#pragma unroll
    for (int n2 = 0; n2 < EMB_WMAX; ++n2) {
      ent[n2] = (n2 < c.N) ? sm[n2] : 0ull;
      if (n2 < n && (uint32_t)(ent[n2] >> 32) == t) leader = false;
    }
    if (!leader) continue;  // the lowest source holding u processes it
    for (int c16 = gl; c16 < c.cps; c16 += G) {
      float g[EPV];
#pragma unroll
      for (int i = 0; i < EPV; ++i) g[i] = 0.f;
#pragma unroll
      for (int n2 = 0; n2 < EMB_WMAX; ++n2) {  // ascending source rank
        if (n2 >= n && n2 < c.N && (uint32_t)(ent[n2] >> 32) == t) {
          const int k2 = (int)(uint32_t)ent[n2];
          float f[EPV];
          if (RAWSRC) {
            const float* src = c.gc_owner + (pn(c, p, n2) * (size_t)c.max_tok + k2) * c.d + c16 * EPV;
#pragma unroll
            for (int i = 0; i < EPV; i += 4) {
              const float4 x = *reinterpret_cast<const float4*>(src + i);
              f[i] = x.x; f[i + 1] = x.y; f[i + 2] = x.z; f[i + 3] = x.w;
            }
          } else {
            Vec<DT>::unpack(ldrow16<true>(recv_of(c, c.r, p, n2) + (size_t)k2 * slice_bytes + (size_t)c16 * 16), f);
          }
#pragma unroll
          for (int i = 0; i < EPV; ++i) g[i] += f[i];
        }
      }
      char* wp = shard + (size_t)u * slice_bytes + (size_t)c16 * 16;
      float w[EPV];
      Vec<DT>::unpack(ld16(wp), w);
      if (c.optim == SGD) {
#pragma unroll
        for (int i = 0; i < EPV; ++i) w[i] = w[i] - c.lr * (c.scale * g[i]);
      } else {
        float* mp = c.adam_m + (size_t)u * c.d + c16 * EPV;
        float* vp = c.adam_v + (size_t)u * c.d + c16 * EPV;
#pragma unroll
        for (int i = 0; i < EPV; i += 4) {
          float4 m4 = *reinterpret_cast<float4*>(mp + i);
          float4 v4 = *reinterpret_cast<float4*>(vp + i);
          float mm[4] = {m4.x, m4.y, m4.z, m4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float gs = c.scale * g[i + j];
            mm[j] = mm[j] + om_b1 * (gs - mm[j]);
            vv[j] = vv[j] + om_b2 * (gs * gs - vv[j]);
            w[i + j] = w[i + j] - alpha * mm[j] / (sqrtf(vv[j]) + c.eps);
          }
          *reinterpret_cast<float4*>(mp + i) = make_float4(mm[0], mm[1], mm[2], mm[3]);
          *reinterpret_cast<float4*>(vp + i) = make_float4(vv[0], vv[1], vv[2], vv[3]);
        }
      }
      st16(wp, Vec<DT>::pack(w));
    }
  }
  if (last_block_done(&c.done_ctr[part ? K_MERGE1 : K_MERGE0])) {
    for (int s = 0; s < c.N; ++s) {
      Flags* f = flags_of(c, s);
      if (part == 0) {
        st_release_sys(&f->prior_done[c.r], t);
        if (c.mode != SPLIT) st_release_sys(&f->def_done[c.r], t);
      } else {
        st_release_sys(&f->def_done[c.r], t);
      }
    }
  }
}

// ------------------------------------------------------------------ launchers
static int bwd_grid(long long warps_of_work, int nsm, int cap_mult) {
  long long blocks = (warps_of_work + (BWD_THREADS / 32) - 1) / (BWD_THREADS / 32);
  if (blocks < 1) blocks = 1;
  if (blocks > (long long)nsm * cap_mult) blocks = (long long)nsm * cap_mult;
  return (int)blocks;
}

template <int DT>
static cudaError_t coal_dispatch(const DevCtx& c, int grid, const void* dY, int p, cudaStream_t s) {
  const int V = (c.cpr + 31) / 32;
  const char* y = static_cast<const char*>(dY);
  if (V <= 1) coal_kernel<DT, 1><<<grid, BWD_THREADS, 0, s>>>(c, y, p);
  else if (V <= 2) coal_kernel<DT, 2><<<grid, BWD_THREADS, 0, s>>>(c, y, p);
  else if (V <= 4) coal_kernel<DT, 4><<<grid, BWD_THREADS, 0, s>>>(c, y, p);
  else if (V <= 8) coal_kernel<DT, 8><<<grid, BWD_THREADS, 0, s>>>(c, y, p);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_coal(const DevCtx& c, const LaunchCfg& L, const void* dY, int p, cudaStream_t s) {
  // one warp per chunk; worst case max_chunks chunks (counts live on the device)
  const int grid = bwd_grid(c.max_chunks, L.nsm, 4);
  return c.dtype == BF16 ? coal_dispatch<BF16>(c, grid, dY, p, s) : coal_dispatch<F32>(c, grid, dY, p, s);
}

cudaError_t launch_defpush(const DevCtx& c, const LaunchCfg& L, int p, cudaStream_t s) {
  const long long work = (long long)c.max_tok * c.cpr;  // upper bound
  int grid = (int)((work + BWD_THREADS * 4 - 1) / (BWD_THREADS * 4));
  if (grid < 1) grid = 1;
  if (grid > L.nsm * 2) grid = L.nsm * 2;
  defpush_kernel<<<grid, BWD_THREADS, 0, s>>>(c, p);
  return cudaGetLastError();
}

cudaError_t launch_rawpush(const DevCtx& c, const LaunchCfg& L, const void* dY, int n, int p, cudaStream_t s) {
  const long long work = (long long)n * c.cpr;
  int grid = (int)((work + BWD_THREADS * 4 - 1) / (BWD_THREADS * 4));
  if (grid < 1) grid = 1;
  if (grid > L.nsm * 2) grid = L.nsm * 2;
  rawpush_kernel<<<grid, BWD_THREADS, 0, s>>>(c, static_cast<const char*>(dY), n, p);
  return cudaGetLastError();
}

template <int DT>
static cudaError_t rawcoal_dispatch(const DevCtx& c, int grid, int p, cudaStream_t s) {
  const int V = (c.cps + 31) / 32;
  if (V <= 1) rawcoal_kernel<DT, 1><<<grid, BWD_THREADS, 0, s>>>(c, p);
  else if (V <= 2) rawcoal_kernel<DT, 2><<<grid, BWD_THREADS, 0, s>>>(c, p);
  else if (V <= 4) rawcoal_kernel<DT, 4><<<grid, BWD_THREADS, 0, s>>>(c, p);
  else if (V <= 8) rawcoal_kernel<DT, 8><<<grid, BWD_THREADS, 0, s>>>(c, p);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_rawcoal(const DevCtx& c, const LaunchCfg& L, int p, cudaStream_t s) {
  const int grid = bwd_grid((long long)c.N * c.max_chunks, L.nsm, 1);  // waits inside: one wave
  return c.dtype == BF16 ? rawcoal_dispatch<BF16>(c, grid, p, s) : rawcoal_dispatch<F32>(c, grid, p, s);
}

cudaError_t launch_merge(const DevCtx& c, const LaunchCfg& L, int p, int part, cudaStream_t s) {
  int G = 1;
  while (G * 2 <= 32 && G * 2 <= c.cps) G *= 2;
  const long long groups = (long long)c.N * c.max_tok;  // upper bound on items
  long long threads = groups * G;
  int grid = (int)((threads + BWD_THREADS - 1) / BWD_THREADS);
  if (grid < 1) grid = 1;
  if (grid > L.nsm) grid = L.nsm;  // waits inside: one wave
  const bool raw = (c.mode == RAW);
  if (c.dtype == BF16) {
    if (raw) merge_kernel<BF16, true><<<grid, BWD_THREADS, 0, s>>>(c, p, part, G);
    else merge_kernel<BF16, false><<<grid, BWD_THREADS, 0, s>>>(c, p, part, G);
  } else {
    if (raw) merge_kernel<F32, true><<<grid, BWD_THREADS, 0, s>>>(c, p, part, G);
    else merge_kernel<F32, false><<<grid, BWD_THREADS, 0, s>>>(c, p, part, G);
  }
  return cudaGetLastError();
}

}  // namespace emb
