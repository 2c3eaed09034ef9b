// k_fwd.cu — forward exchange and next-batch prefetch (a5).
//
// PAPER.md:280 (§4.1.3): "embedding in each process firstly looks up all
// training data of this step and produces a different embedding result.  Then
// AlltoAll is called for redistributing the embedding results so that each
// process gets one embedding result minibatch".  Fig. 3 caption.
//
// B200 design: the AlltoAll + column concat is done as
// ONE pull kernel.  Rank r reads, for every token j of its own minibatch and
// every owner s, the 16-byte vectors of shard_s[ids[j], :] straight out of
// s's HBM over NVLink (CUDA IPC mapping) and stores them at their final column
// offset s*d of out[j, :].  No send/recv staging, no unpack kernel, and the
// forward needs no id all-gather (only the owners' "prior part applied" flags).
// The all-gather of the ids (Alg. 1's "gathered training data")
// still happens here when it was not prefetched, because the backward routing
// of every rank needs every rank's ids.
#include "kernels.cuh"

namespace emb {

static constexpr int FWD_THREADS = 512;
static constexpr int FWD_UNROLL = 4;

__global__ void __launch_bounds__(FWD_THREADS) fwd_kernel(DevCtx c, const int* __restrict__ ids, int n,
                                                          char* __restrict__ out, int p, int prefetched) {
  const uint32_t t = c.t_rec[p ^ 1] + 1;  // iteration number (device-resident, graph-replay safe)
  if (blockIdx.x == 0 && threadIdx.x == 0) c.t_rec[p] = t;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;

  // (a1) all-gather of this rank's ids into every peer's gids[p][r]
  if (!prefetched) {
    for (int i = tid; i < n * c.N; i += nth) {
      const int s = i / n, j = i - s * n;
      gids_of(c, s, p, c.r)[j] = ids[j];
    }
    if (tid < c.N) *ntok_of(c, tid, p, c.r) = n;
    if (last_block_done(&c.done_ctr[K_FWD_IDS])) {
      for (int s = 0; s < c.N; ++s) {
        st_release_sys(&flags_of(c, s)->ids[c.r], t);
        atomicAdd(&c.stats[2 * c.N + s], (unsigned long long)n * 4ull);
      }
    }
  } else {
    // prefetched by backward(t-1): the ids must be the promised next_ids
    const int* mine = gids_of(c, c.r, p, c.r);
    for (int j = tid; j < n; j += nth)
      if (mine[j] != ids[j]) atomicOr(c.err, ERR_STATE);
    if (tid == 0 && *ntok_of(c, c.r, p, c.r) != n) atomicOr(c.err, ERR_STATE);
  }

  // wait: every owner applied the prior part of t-1 and the scheduled part of t-2
  if (threadIdx.x == 0) {
    Flags* f = flags_of(c, c.r);
    for (int s = 0; s < c.N; ++s) {
      wait_flag(c, &f->prior_done[s], t - 1);
      wait_flag(c, &f->def_done[s], t - 2);
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int s = 0; s < c.N; ++s) atomicAdd(&c.stats[s], (unsigned long long)n * c.d * c.esz);

  // (a2-a4) pull-gather: 16-byte chunk q of out = row j, column chunk cc;
  // cc lies in owner s = cc / cps's slice.
  const size_t total = (size_t)n * c.cpr;
  const size_t slice_bytes = (size_t)c.d * c.esz;
  for (size_t q0 = tid; q0 < total; q0 += (size_t)nth * FWD_UNROLL) {
    uint4 v[FWD_UNROLL];
#pragma unroll
    for (int u = 0; u < FWD_UNROLL; ++u) {
      const size_t q = q0 + (size_t)u * nth;
      v[u] = make_uint4(0, 0, 0, 0);
      if (q < total) {
        const int j = (int)(q / c.cpr);
        const int cc = (int)(q - (size_t)j * c.cpr);
        const int s = cc / c.cps, cs = cc - s * c.cps;
        const int id = __ldg(ids + j);
        if ((unsigned)id < (unsigned long long)c.L) {
          v[u] = ld16_nc(shard_of(c, s) + (size_t)id * slice_bytes + (size_t)cs * 16);
        } else if (cs == 0) {
          atomicOr(c.err, ERR_ID);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < FWD_UNROLL; ++u) {
      const size_t q = q0 + (size_t)u * nth;
      if (q < total) st16(out + q * 16, v[u]);
    }
  }
}

// a5: next-batch prefetch.  Push next ids to every peer (gids[p^1][r]); with
// do_mark (SPLIT), wait for every rank's next ids and tag D_next:
// nextmark[id] = t+1  (no clearing ever needed — epoch tags).
__global__ void __launch_bounds__(256) ids_kernel(DevCtx c, const int* __restrict__ next_ids, int n_next,
                                                  int p, int do_mark) {
  const uint32_t t = c.t_rec[p];
  const int p1 = p ^ 1;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;
  if (next_ids != nullptr) {
    for (int i = tid; i < n_next * c.N; i += nth) {
      const int s = i / n_next, j = i - s * n_next;
      gids_of(c, s, p1, c.r)[j] = next_ids[j];
    }
    if (tid < c.N) *ntok_of(c, tid, p1, c.r) = n_next;
    if (last_block_done(&c.done_ctr[K_IDS])) {
      for (int s = 0; s < c.N; ++s) {
        st_release_sys(&flags_of(c, s)->ids[c.r], t + 1);
        atomicAdd(&c.stats[2 * c.N + s], (unsigned long long)n_next * 4ull);
      }
    }
  }
  if (!do_mark) return;
  block_wait_all(c, flags_of(c, c.r)->ids, t + 1);  // all blocks co-resident (grid <= #SM)
  for (int n = 0; n < c.N; ++n) {
    const int cnt = __ldcg(ntok_of(c, c.r, p1, n));   // peer-written: read at L2
    const int* g = gids_of(c, c.r, p1, n);
    for (int j = tid; j < cnt; j += nth) {
      const int id = __ldcg(g + j);
      if ((unsigned)id < (unsigned long long)c.L) c.nextmark[id] = (int)(t + 1);
    }
  }
}

cudaError_t launch_fwd(const DevCtx& c, const LaunchCfg& L, const int* ids, int n, void* out, int p,
                       int prefetched, cudaStream_t s) {
  long long work = (long long)n * c.cpr;
  int grid = (int)((work + (long long)FWD_THREADS * FWD_UNROLL - 1) / ((long long)FWD_THREADS * FWD_UNROLL));
  if (grid < 1) grid = 1;
  if (grid > L.nsm) grid = L.nsm;  // waits inside: keep one wave
  fwd_kernel<<<grid, FWD_THREADS, 0, s>>>(c, ids, n, static_cast<char*>(out), p, prefetched);
  return cudaGetLastError();
}

cudaError_t launch_ids(const DevCtx& c, const LaunchCfg& L, const int* next_ids, int n_next, int p, int do_mark,
                       cudaStream_t s) {
  long long work = (long long)c.N * (next_ids ? n_next : 0) + (long long)c.N * c.max_tok;
  int grid = (int)((work + 4095) / 4096);
  if (grid < 1) grid = 1;
  if (grid > L.nsm) grid = L.nsm;
  ids_kernel<<<grid, 256, 0, s>>>(c, next_ids, n_next, p, do_mark);
  return cudaGetLastError();
}

}  // namespace emb
