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
// B200 design.  Rows are addressed by the sender's
// unique index i (ascending unique ids from the sort); the prior / scheduled
// class of a row is the D_next mark of its id.
//   coal_reduce  sender-side segmented reduce of dY in fp32, one warp per
//            reduce chunk of <= C rows of one unique, ascending positions; a
//            single-chunk unique's sum goes to gcoal, a multi-chunk (Zipf-head)
//            unique's chunk sums to scratch (no float atomics).
//   coal_apply   Zipf-head partials combined per (unique, column slice) in a
//            fixed order (deterministic); then per coalesced row and 16-byte
//            chunk:
//              N == 1  optimizer step applied in place (one source = the
//                      merged gradient: no exchange, no merge kernel);
//              N > 1   rounded to the wire dtype and stored straight into the
//                      owner's receive row i over NVLink (prior rows), or into
//                      the local stage (scheduled rows) — COALESCE +
//                      INDEX_SELECT + AlltoAll in one pass.
//   defpush  pushes the staged scheduled rows (side stream, lowest priority).
//   rawpush / rawcoal   RAW mode: raw dY slices travel, the owner coalesces
//            every source (fp32, no wire rounding).
//   merge    owner: each row's contributions summed in ascending source rank
//            (fp32), scaled, fused SGD / Adam update of shard, m, v.
#include <stddef.h>

#include "kernels.cuh"

namespace emb {

static constexpr int BWD_THREADS = 256;
static constexpr int BWD_WARPS = BWD_THREADS / 32;

// Rows in flight per warp in the segmented reduce.  Most uniques have 1-2 rows
// (Zipf tail), so 2 in flight costs little latency and saves load registers.
#ifndef EMB_RB
#define EMB_RB 4
#endif

// acc[v*EPV + i] = sum over rows perm[b..e) (ascending) of row[c16 = lane + 32 v]
template <int DT, int V, bool PEER>
__device__ __forceinline__ void reduce_rows(const char* __restrict__ base, size_t stride, int ncol16,
                                            const int* __restrict__ perm, int b, int e, float* acc, int pos1 = -1) {
  constexpr int EPV = Vec<DT>::EPV;
  constexpr int RB = EMB_RB;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < V * EPV; ++i) acc[i] = 0.f;
  static_assert(32 % RB == 0, "row batches must tile the 32-position windows");
  int mypos = 0;  // lane j holds perm[window + j]: one load per 32 rows, not one per row batch
  for (int i = b; i < e; i += RB) {
    if (((i - b) & 31) == 0) {
      const int j = i + lane;
      mypos = (pos1 >= 0) ? pos1 : ((j < e) ? __ldg(perm + j) : 0);  // pos1: a single-row chunk's position
    }
    int pos[RB];
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) pos[rr] = __shfl_sync(0xffffffffu, mypos, (i - b + rr) & 31);
    uint4 buf[RB][V];
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      if (i + rr < e) {
        const char* row = base + (size_t)pos[rr] * stride;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int c16 = lane + 32 * v;
          if (c16 < ncol16) buf[rr][v] = PEER ? ld16_cg(row + (size_t)c16 * 16) : ld16_nc(row + (size_t)c16 * 16);
        }
      }
    }
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
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

// fp32 partial rows: lane's chunk c16 holds floats [c16*EPV, c16*EPV+EPV)
template <int EPV, int V>
__device__ __forceinline__ void store_partial(float* dst, int ncol16, const float* acc) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int c16 = lane + 32 * v;
    if (c16 < ncol16) {
#pragma unroll
      for (int q = 0; q < EPV; q += 4)
        *reinterpret_cast<float4*>(dst + c16 * EPV + q) =
            make_float4(acc[v * EPV + q], acc[v * EPV + q + 1], acc[v * EPV + q + 2], acc[v * EPV + q + 3]);
    }
  }
}

// Sum partial rows [q0, q1) (ascending) into acc.
template <int EPV, int V>
__device__ __forceinline__ void sum_partials(const float* base, int dw, int ncol16, int q0, int q1, float* acc) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < V * EPV; ++i) acc[i] = 0.f;
  constexpr int PB = 8 / EPV;  // partial rows in flight: 32 registers of loads whatever the dtype
  for (int q = q0; q < q1; q += PB) {
    float4 buf[PB][V][EPV / 4];
#pragma unroll
    for (int rr = 0; rr < PB; ++rr)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int c16 = lane + 32 * v;
        if (q + rr < q1 && c16 < ncol16)
#pragma unroll
          for (int x = 0; x < EPV / 4; ++x)
            buf[rr][v][x] = __ldcg(reinterpret_cast<const float4*>(base + (size_t)(q + rr) * dw + c16 * EPV) + x);
      }
#pragma unroll
    for (int rr = 0; rr < PB; ++rr)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int c16 = lane + 32 * v;
        if (q + rr < q1 && c16 < ncol16)
#pragma unroll
          for (int x = 0; x < EPV / 4; ++x) {
            acc[v * EPV + 4 * x + 0] += buf[rr][v][x].x;
            acc[v * EPV + 4 * x + 1] += buf[rr][v][x].y;
            acc[v * EPV + 4 * x + 2] += buf[rr][v][x].z;
            acc[v * EPV + 4 * x + 3] += buf[rr][v][x].w;
          }
      }
  }
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Sparse optimizer math on EPV elements of one row chunk; g = merged, unscaled
// gradient.  SGD: w -= lr*g.  Adam (PyTorch SparseAdam form, step t folded
// into alpha_t, readings R3/R4): m += (1-b1)(g-m); v += (1-b2)(g^2-v);
// w -= alpha_t m / (sqrt(v)+eps).  Adagrad (PAPER.md:594
// names it among the element-wise sparse optimizers; PyTorch Adagrad form with
// lr_decay 0, initial accumulator 0): s += g^2; w -= lr g / (sqrt(s)+eps), the
// accumulator s kept in the first-moment buffer.  sqrt / reciprocal use the
// SFU (MUFU) approximations: relative error ~1e-7, far inside the 1e-5 parity
// bound, where an IEEE div+sqrt would cost ~30 instructions per element.
template <int EPV>
__device__ __forceinline__ void opt_math(const DevCtx& c, float alpha, const float* g, float* w, float* mm, float* vv) {
  if (c.optim == SGD) {
#pragma unroll
    for (int i = 0; i < EPV; ++i) w[i] = w[i] - c.lr * (c.scale * g[i]);
    return;
  }
  if (c.optim == ADAGRAD) {
#pragma unroll
    for (int i = 0; i < EPV; ++i) {
      const float gs = c.scale * g[i];
      mm[i] = mm[i] + gs * gs;
      w[i] = w[i] - c.lr * gs * rcp_approx(sqrt_approx(mm[i]) + c.eps);
    }
    return;
  }
  const float om_b1 = 1.f - c.beta1, om_b2 = 1.f - c.beta2;
#pragma unroll
  for (int i = 0; i < EPV; ++i) {
    const float gs = c.scale * g[i];
    mm[i] = mm[i] + om_b1 * (gs - mm[i]);
    vv[i] = vv[i] + om_b2 * (gs * gs - vv[i]);
    w[i] = w[i] - alpha * mm[i] * rcp_approx(sqrt_approx(vv[i]) + c.eps);
  }
}

// ------------------------------------------------------------------ sender coalesce
// Two kernels, so that neither needs a CTA barrier on its hot loop:
//  coal_reduce  warp per reduce chunk (<= C rows of one unique, ascending
//               position), fp32 sums in registers: a single-chunk unique's sum
//               goes to gcoal[i], a multi-chunk (Zipf-head) unique's chunk sums
//               to scratch.  No shared memory, no barriers: the occupancy is
//               what hides the perm -> dY load chain.
//  coal_apply   (1) CTA per multi-chunk unique: its chunk sums are combined in
//               a fixed order (warps sum contiguous ranges, then a fixed warp-
//               order shared-memory sum: deterministic) and emitted by the
//               CTA; (2) thread per (single-chunk unique, 16-byte wire chunk):
//               N == 1 the optimizer step in place (one source = the merged
//               gradient), N > 1 the wire-rounded slice stored into the
//               owner's receive row i over NVLink (prior) or the stage
//               (scheduled).  Every load of an item is issued before its math.
template <int DT, int V>
__global__ void __launch_bounds__(BWD_THREADS) coal_reduce_kernel(DevCtx c, const char* __restrict__ dY, int p,
                                                                  int gate_flags) {
  EMB_TR_ENTRY();
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  constexpr int EPV = Vec<DT>::EPV;
  const int r = c.r;
  const uint32_t t = c.t_rec[p];
  (void)t;
  EMB_TR_BEGIN(3, t);
  EMB_TR_WAITED(3, t);
  const int NCH = counts_of(c, p, r)[CNT_NCH];
  const int4* desc = c.chunk_desc + pn(c, p, r) * (size_t)c.max_chunks;
  const int* perm = c.perm + pn(c, p, r) * (size_t)c.max_tok;
  float* part = c.scratch + (size_t)p * c.max_chunks * c.D;
  const size_t row_bytes = (size_t)c.D * c.esz;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int ch = gw; ch < NCH; ch += nw) {
    const int4 dsc = desc[ch];  // {unique i, perm begin, perm end, chunks of i}
    if (c.bypass && desc_pos1(dsc.w) >= 0) continue;  // single-row unique: the apply reads its dY row
    float acc[V * EPV];
    reduce_rows<DT, V, false>(dY, row_bytes, c.cpr, perm, dsc.y, dsc.z, acc, desc_pos1(dsc.w));
    store_partial<EPV, V>((desc_nch(dsc.w) > 1) ? part + (size_t)ch * c.D : c.gcoal + (size_t)dsc.x * c.D, c.cpr,
                          acc);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // gate duties folded into this kernel's CTA 0 (no gate kernel before the
    // apply): bit 0, N == 1 prefetch check (fingerprints of fwd(t) and sort(t));
    // bit 1, SPLIT N > 1: the D_next tags of t+1 (marktag, aux) are complete
    if (gate_flags & 1) {
      unsigned* f = c.fp + p * 4;
      if (__ldcg(f) != __ldcg(f + 2) || __ldcg(f + 1) != __ldcg(f + 3)) atomicOr(c.err, ERR_STATE);
      f[0] = f[1] = f[2] = f[3] = 0;
    }
    if (gate_flags & 2) wait_local(c, c.marked + p, t, 8 * 16 + 1);
  }
  EMB_TR_END(3, t);
  pdl_trigger();
}

#ifndef EMB_APPLY_EA_F32
#define EMB_APPLY_EA_F32 2
#endif
#ifndef EMB_APPLY_EA_BF16
#define EMB_APPLY_EA_BF16 1
#endif
#define EMB_APPLY_EA(EPV) ((EPV) == 4 ? EMB_APPLY_EA_F32 : EMB_APPLY_EA_BF16)  // single-chunk rows in flight per thread
#ifndef EMB_APPLY_GRID_PER_SM
#define EMB_APPLY_GRID_PER_SM 8  // grid cap (the grid is sized from max_tok: U lives on the device)
#endif
#ifndef EMB_APPLY_MINB
#define EMB_APPLY_MINB 4  // measured: 3 -> 4 resident CTAs per SM, LM N=1 23.3 -> 22.0 us
#endif
// One 16-byte wire chunk c16 of coalesced row k (id, merged fp32 g): loads of
// the state first (apply_load), then the math and stores (apply_store).
//   N == 1: optimizer step in place (SGD / Adam, opt_math);
//   N > 1:  the wire-rounded slice goes to the owner's receive row k (prior,
//           NVLink store) or to the stage (scheduled).
template <int DT>
struct ApplyState {
  uint4 w;
  float m[Vec<DT>::EPV], v[Vec<DT>::EPV];
};
template <int DT>
__device__ __forceinline__ void apply_load(const DevCtx& c, int id, int c16, ApplyState<DT>& st) {
  constexpr int EPV = Vec<DT>::EPV;
  if (c.N != 1) return;
  const size_t u = (size_t)id;
  st.w = ld16(shard_of(c, c.r) + u * ((size_t)c.d * c.esz) + (size_t)c16 * 16);
  if (c.optim != SGD) {  // Adam m, v; Adagrad accumulator (in m)
#pragma unroll
    for (int x = 0; x < EPV; x += 4) {
      const float4 m4 = *reinterpret_cast<const float4*>(c.adam_m + u * c.d + c16 * EPV + x);
      st.m[x] = m4.x; st.m[x + 1] = m4.y; st.m[x + 2] = m4.z; st.m[x + 3] = m4.w;
      if (c.optim == ADAM) {
        const float4 v4 = *reinterpret_cast<const float4*>(c.adam_v + u * c.d + c16 * EPV + x);
        st.v[x] = v4.x; st.v[x + 1] = v4.y; st.v[x + 2] = v4.z; st.v[x + 3] = v4.w;
      }
    }
  }
}
template <int DT>
__device__ __forceinline__ void apply_store(const DevCtx& c, int p, uint32_t t, int k, int id, int c16, const float* g,
                                            ApplyState<DT>& st, float alpha) {
  constexpr int EPV = Vec<DT>::EPV;
  const uint4 gw = Vec<DT>::pack(g);  // wire rounding point (reading R11)
  const size_t slice_bytes = (size_t)c.d * c.esz;
  if (c.N == 1) {
    const size_t u = (size_t)id;
    float gr[EPV], wv[EPV];
    Vec<DT>::unpack(gw, gr);
    Vec<DT>::unpack(st.w, wv);
    opt_math<EPV>(c, alpha, gr, wv, st.m, st.v);
    st16(shard_of(c, c.r) + u * slice_bytes + (size_t)c16 * 16, Vec<DT>::pack(wv));
    if (c.optim != SGD) {
#pragma unroll
      for (int x = 0; x < EPV; x += 4) {
        *reinterpret_cast<float4*>(c.adam_m + u * c.d + c16 * EPV + x) =
            make_float4(st.m[x], st.m[x + 1], st.m[x + 2], st.m[x + 3]);
        if (c.optim == ADAM)
          *reinterpret_cast<float4*>(c.adam_v + u * c.d + c16 * EPV + x) =
              make_float4(st.v[x], st.v[x + 1], st.v[x + 2], st.v[x + 3]);
      }
    }
  } else if (is_prior(c, p, t, id)) {
    const int s = c16 / c.cps, cs = c16 - s * c.cps;
    st16(recv_of(c, s, p, c.r) + (size_t)k * slice_bytes + (size_t)cs * 16, gw);
  } else {
    st16(c.stage + ((size_t)p * c.max_tok + k) * ((size_t)c.D * c.esz) + (size_t)c16 * 16, gw);
  }
}

static constexpr int SLICE = 128;  // fp32 columns per combine slice (one float4 per lane)

template <int DT>
__global__ void __launch_bounds__(BWD_THREADS, EMB_APPLY_MINB) coal_apply_kernel(DevCtx c, const char* __restrict__ dY,
                                                                                 int p) {
  EMB_TR_ENTRY();
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  constexpr int EPV = Vec<DT>::EPV;
  __shared__ __align__(16) float comb[BWD_WARPS][SLICE];  // warp partial sums of one column slice
  __shared__ __align__(16) float row[SLICE];              // combined slice
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = c.r;
  const uint32_t t = c.t_rec[p];
  EMB_TR_BEGIN(16, t);
  EMB_TR_WAITED(16, t);
  const int* cnt = counts_of(c, p, r);
  const int U = cnt[CNT_U], NLONG = cnt[CNT_NLONG];
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int s = 0; s < c.N; ++s) atomicAdd(&c.stats[c.N + s], (unsigned long long)U * c.d * c.esz);
  const float alpha = (c.optim == ADAM) ? c.alpha[p] : 0.f;
  const size_t bpn = pn(c, p, r) * (size_t)c.max_tok;
  const int* uid = c.uid + bpn;
  const int* chunk_off = c.chunk_off + pn(c, p, r) * (size_t)(c.max_tok + 1);
  const int* upos = c.upos + bpn;
  const int* long_u = c.long_u + pn(c, p, r) * (size_t)c.max_long;
  const float* part = c.scratch + (size_t)p * c.max_chunks * c.D;

  // (1) multi-chunk (Zipf-head) uniques, split into (unique, 128-column slice)
  //     items so that a huge segment (e.g. the pad id) is combined by many
  //     CTAs: warps sum contiguous ranges of chunk partials (ascending, 8 loads
  //     in flight), then a fixed warp-order sum — deterministic.
  const int NS = (c.D + SLICE - 1) / SLICE;
  for (int item = blockIdx.x; item < NLONG * NS; item += gridDim.x) {
    const int lu = item / NS, sl = item - lu * NS;
    const int kk = long_u[lu];
    const int c0 = chunk_off[kk], n2 = chunk_off[kk + 1] - c0;
    const int q0 = c0 + (int)((long long)n2 * w / BWD_WARPS), q1 = c0 + (int)((long long)n2 * (w + 1) / BWD_WARPS);
    const int col = sl * SLICE + lane * 4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (col < c.D) {
      for (int q = q0; q < q1; q += 8) {
        float4 b[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          b[j] = (q + j < q1) ? __ldcg(reinterpret_cast<const float4*>(part + (size_t)(q + j) * c.D + col))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc.x += b[j].x; acc.y += b[j].y; acc.z += b[j].z; acc.w += b[j].w;
        }
      }
    }
    *reinterpret_cast<float4*>(&comb[w][lane * 4]) = acc;
    __syncthreads();
    if (threadIdx.x < SLICE) {
      float sum = 0.f;
#pragma unroll
      for (int ww = 0; ww < BWD_WARPS; ++ww) sum += comb[ww][threadIdx.x];
      row[threadIdx.x] = sum;
    }
    __syncthreads();
    if (threadIdx.x < SLICE / EPV) {
      const int c16 = sl * (SLICE / EPV) + threadIdx.x;
      if (c16 < c.cpr) {
        const int id = uid[kk];
        ApplyState<DT> st;
        apply_load<DT>(c, id, c16, st);
        float g[EPV];
#pragma unroll
        for (int x = 0; x < EPV; ++x) g[x] = row[threadIdx.x * EPV + x];
        apply_store<DT>(c, p, t, kk, id, c16, g, st, alpha);
      }
    }
    __syncthreads();
  }

  // (2) single-chunk uniques: RPB rows per CTA pass, thread = one 16-byte wire
  //     chunk (the (row, chunk) split is computed once: no division in the loop)
  constexpr int EA = EMB_APPLY_EA(EPV);  // rows in flight per thread
  const int RPB = BWD_THREADS / c.cpr;
  const int rl = threadIdx.x / c.cpr, c16 = threadIdx.x - rl * c.cpr;
  if (rl < RPB) {
    const int step = gridDim.x * RPB;
    for (int k0 = blockIdx.x * RPB + rl; k0 < U; k0 += step * EA) {
      int kk[EA], id[EA], up[EA];
      bool ok[EA];
      float g[EA][EPV];
      ApplyState<DT> st[EA];
#pragma unroll
      for (int j = 0; j < EA; ++j) {
        kk[j] = k0 + j * step;
        // uid and chunk_off loads issued together (uid[k] is valid for every k < U)
        const bool in = kk[j] < U;
        id[j] = in ? __ldcg(uid + kk[j]) : 0;
        up[j] = (in && c.bypass) ? __ldcg(upos + kk[j]) : -1;
        ok[j] = in && (__ldcg(chunk_off + kk[j] + 1) - __ldcg(chunk_off + kk[j])) == 1;
      }
#pragma unroll
      for (int j = 0; j < EA; ++j) {
        if (!ok[j]) continue;
        if (up[j] >= 0) {  // single-row unique: its sum is its dY row (exact in fp32)
          Vec<DT>::unpack(ld16_nc(dY + (size_t)up[j] * ((size_t)c.D * c.esz) + (size_t)c16 * 16), g[j]);
        } else {
          const float* gp = c.gcoal + (size_t)kk[j] * c.D + c16 * EPV;
#pragma unroll
          for (int x = 0; x < EPV; x += 4) {
            const float4 g4 = __ldcg(reinterpret_cast<const float4*>(gp + x));
            g[j][x] = g4.x; g[j][x + 1] = g4.y; g[j][x + 2] = g4.z; g[j][x + 3] = g4.w;
          }
        }
        apply_load<DT>(c, id[j], c16, st[j]);
      }
#pragma unroll
      for (int j = 0; j < EA; ++j)
        if (ok[j]) apply_store<DT>(c, p, t, kk[j], id[j], c16, g[j], st[j], alpha);
    }
  }
  EMB_TR_END(16, t);
  pdl_trigger();
}

// ------------------------------------------------------------------ scheduled push (N > 1)
__global__ void __launch_bounds__(BWD_THREADS) defpush_kernel(DevCtx c, int p) {
  EMB_TR_ENTRY();
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  const int r = c.r;
  const uint32_t t = c.t_rec[p];
  EMB_TR_BEGIN(5, t);
  EMB_TR_WAITED(5, t);
  const int U = counts_of(c, p, r)[CNT_U];
  const int* uid = c.uid + pn(c, p, r) * (size_t)c.max_tok;
  const size_t row_bytes = (size_t)c.D * c.esz, slice_bytes = (size_t)c.d * c.esz;
  const size_t total = (size_t)U * c.cpr;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (size_t q = tid; q < total; q += nth) {
    const int k = (int)(q / c.cpr), c16 = (int)(q - (size_t)k * c.cpr);
    if (is_prior(c, p, t, uid[k])) continue;  // prior rows went out with the coalesce
    const uint4 val = ld16_nc(c.stage + ((size_t)p * c.max_tok + k) * row_bytes + (size_t)c16 * 16);
    const int s = c16 / c.cps, cs = c16 - s * c.cps;
    st16(recv_of(c, s, p, r) + (size_t)k * slice_bytes + (size_t)cs * 16, val);
  }
  EMB_TR_END(5, t);
  pdl_trigger();
}

// ------------------------------------------------------------------ RAW mode
__global__ void __launch_bounds__(BWD_THREADS) rawpush_kernel(DevCtx c, const char* __restrict__ dY, int n, int p) {
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  const int r = c.r;
  const size_t row_bytes = (size_t)c.D * c.esz, slice_bytes = (size_t)c.d * c.esz;
  const size_t total = (size_t)n * c.cpr;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  if (tid == 0)
    for (int s = 0; s < c.N; ++s) atomicAdd(&c.stats[c.N + s], (unsigned long long)n * slice_bytes);
  for (size_t q = tid; q < total; q += nth) {
    const int j = (int)(q / c.cpr), c16 = (int)(q - (size_t)j * c.cpr);
    const uint4 val = ld16_nc(dY + (size_t)j * row_bytes + (size_t)c16 * 16);
    const int s = c16 / c.cps, cs = c16 - s * c.cps;
    st16(recv_of(c, s, p, r) + (size_t)j * slice_bytes + (size_t)cs * 16, val);
  }
  pdl_trigger();
}

// owner-side coalesce of every source's raw slices -> gc_owner[n][i] (fp32)
template <int DT, int V>
__global__ void __launch_bounds__(BWD_THREADS) rawcoal_a_kernel(DevCtx c, int p) {
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  constexpr int EPV = Vec<DT>::EPV;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t t = c.t_rec[p];
  (void)t;  // N > 1: every rawpush completed (the gate before this kernel waited for the pub flags)
  int nchs[EMB_WMAX];
  int total = 0;
#pragma unroll
  for (int n = 0; n < EMB_WMAX; ++n) {
    nchs[n] = (n < c.N) ? counts_of(c, p, n)[CNT_NCH] : 0;
    total += nchs[n];
  }
  const size_t slice_bytes = (size_t)c.d * c.esz;
  float acc[V * EPV];
  for (int gch = gw; gch < total; gch += nw) {
    int n = 0, ch = gch;
#pragma unroll
    for (int m = 0; m < EMB_WMAX - 1; ++m)
      if (n == m && ch >= nchs[m]) { ch -= nchs[m]; n = m + 1; }
    const size_t bpn = pn(c, p, n) * (size_t)c.max_tok;
    const int4 dsc = c.chunk_desc[pn(c, p, n) * (size_t)c.max_chunks + ch];  // {k, begin, end, nch}
    const int k = dsc.x, nch = desc_nch(dsc.w);
    reduce_rows<DT, V, true>(recv_of(c, c.r, p, n), slice_bytes, c.cps, c.perm + bpn, dsc.y, dsc.z, acc);
    float* dst = (nch > 1) ? c.scratch + (size_t)p * c.max_chunks * c.D + ((size_t)n * c.max_chunks + ch) * c.d
                           : c.gc_owner + (bpn + k) * (size_t)c.d;
    store_partial<EPV, V>(dst, c.cps, acc);
  }
  pdl_trigger();
}

template <int DT, int V>
__global__ void __launch_bounds__(BWD_THREADS) rawcoal_b_kernel(DevCtx c, int p) {
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  constexpr int EPV = Vec<DT>::EPV;
  extern __shared__ __align__(16) float wpart[];  // [BWD_WARPS][d]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int nls[EMB_WMAX];
  int total = 0;
#pragma unroll
  for (int n = 0; n < EMB_WMAX; ++n) {
    nls[n] = (n < c.N) ? counts_of(c, p, n)[CNT_NLONG] : 0;
    total += nls[n];
  }
  float acc[V * EPV];
  for (int gl = blockIdx.x; gl < total; gl += gridDim.x) {
    int n = 0, li = gl;
#pragma unroll
    for (int m = 0; m < EMB_WMAX - 1; ++m)
      if (n == m && li >= nls[m]) { li -= nls[m]; n = m + 1; }
    const size_t bpn = pn(c, p, n) * (size_t)c.max_tok;
    const int k = c.long_u[pn(c, p, n) * (size_t)c.max_long + li];
    const int* chunk_off = c.chunk_off + pn(c, p, n) * (size_t)(c.max_tok + 1);
    const int c0 = chunk_off[k], nch = chunk_off[k + 1] - c0;
    const int q0 = c0 + (int)((long long)nch * w / BWD_WARPS), q1 = c0 + (int)((long long)nch * (w + 1) / BWD_WARPS);
    sum_partials<EPV, V>(c.scratch + (size_t)p * c.max_chunks * c.D + (size_t)n * c.max_chunks * c.d, c.d, c.cps, q0,
                         q1, acc);
    store_partial<EPV, V>(wpart + (size_t)w * c.d, c.cps, acc);
    __syncthreads();
    if (w == 0) {
#pragma unroll
      for (int i = 0; i < V * EPV; ++i) acc[i] = 0.f;
      for (int ww = 0; ww < BWD_WARPS; ++ww)
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int c16 = lane + 32 * v;
          if (c16 < c.cps)
#pragma unroll
            for (int i = 0; i < EPV; ++i) acc[v * EPV + i] += wpart[(size_t)ww * c.d + c16 * EPV + i];
        }
      store_partial<EPV, V>(c.gc_owner + (bpn + k) * (size_t)c.d, c.cps, acc);
    }
    __syncthreads();
  }
  pdl_trigger();
}

// ------------------------------------------------------------------ owner merge + update
// Items: every (source n, unique i) of the requested part (part 0: prior, or
// everything outside SPLIT; part 1: scheduled).  The lowest source holding an
// id (slotmap tag == t) applies it: contributions of all sources holding it
// are summed in ascending source rank, then scaled and applied.
template <int DT, bool RAWSRC>
__global__ void __launch_bounds__(BWD_THREADS) merge_kernel(DevCtx c, int p, int part, int G) {
  EMB_TR_ENTRY();
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  constexpr int EPV = Vec<DT>::EPV;
  const uint32_t t = c.t_rec[p];
  (void)t;
  EMB_TR_BEGIN(part ? 6 : 4, t);
  EMB_TR_WAITED(part ? 6 : 4, t);
  // N > 1: every sender's pass of this part completed (the gate before this
  // kernel waited for their pub flags).  Items: this part's plan entries (one
  // per distinct id: the id and its unique index at every source, plan_kernel).
  // N == 1 (RAW mode only): one source, every unique is its own leader
  const int total = (c.N == 1) ? counts_of(c, p, 0)[CNT_U] : c.plan_cnt[p * 2 + part];
  const int PW = 1 + c.N;
  const int* plan = (c.N == 1) ? nullptr : c.plan + ((size_t)p * 2 + part) * c.N * c.max_tok * PW;
  const float alpha = (c.optim == ADAM) ? c.alpha[p] : 0.f;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int grp = gtid / G, gl = gtid - grp * G, ngrp = (gridDim.x * blockDim.x) / G;
  const size_t slice_bytes = (size_t)c.d * c.esz;
  char* shard = shard_of(c, c.r);
  for (int item = grp; item < total; item += ngrp) {
    int u, ks[EMB_WMAX];
    if (c.N == 1) {
      u = c.uid[pn(c, p, 0) * (size_t)c.max_tok + item];
      ks[0] = item;
#pragma unroll
      for (int n2 = 1; n2 < EMB_WMAX; ++n2) ks[n2] = -1;
    } else {
      const int* e = plan + (size_t)item * PW;
      u = e[0];
#pragma unroll
      for (int n2 = 0; n2 < EMB_WMAX; ++n2) ks[n2] = (n2 < c.N) ? e[1 + n2] : -1;
    }
    for (int c16 = gl; c16 < c.cps; c16 += G) {
      // state loads first (independent of the contributions)
      char* wp = shard + (size_t)u * slice_bytes + (size_t)c16 * 16;
      const uint4 wraw = ld16(wp);
      float mm[EPV], vv[EPV];
      float* mp = c.adam_m + (size_t)u * c.d + c16 * EPV;
      float* vp = c.adam_v + (size_t)u * c.d + c16 * EPV;
      if (c.optim != SGD) {
#pragma unroll
        for (int i = 0; i < EPV; i += 4) {
          const float4 m4 = *reinterpret_cast<const float4*>(mp + i);
          mm[i] = m4.x; mm[i + 1] = m4.y; mm[i + 2] = m4.z; mm[i + 3] = m4.w;
          if (c.optim == ADAM) {
            const float4 v4 = *reinterpret_cast<const float4*>(vp + i);
            vv[i] = v4.x; vv[i + 1] = v4.y; vv[i + 2] = v4.z; vv[i + 3] = v4.w;
          }
        }
      }
      float g[EPV];
#pragma unroll
      for (int i = 0; i < EPV; ++i) g[i] = 0.f;
#pragma unroll
      for (int n2 = 0; n2 < EMB_WMAX; ++n2) {  // ascending source rank (reading R12)
        if (ks[n2] >= 0) {
          const int k2 = ks[n2];
          float f[EPV];
          if (RAWSRC) {
            const float* src = c.gc_owner + (pn(c, p, n2) * (size_t)c.max_tok + k2) * c.d + c16 * EPV;
#pragma unroll
            for (int i = 0; i < EPV; i += 4) {
              const float4 x = __ldcg(reinterpret_cast<const float4*>(src + i));
              f[i] = x.x; f[i + 1] = x.y; f[i + 2] = x.z; f[i + 3] = x.w;
            }
          } else {
            Vec<DT>::unpack(ld16_cg(recv_of(c, c.r, p, n2) + (size_t)k2 * slice_bytes + (size_t)c16 * 16), f);
          }
#pragma unroll
          for (int i = 0; i < EPV; ++i) g[i] += f[i];
        }
      }
      float w[EPV];
      Vec<DT>::unpack(wraw, w);
      opt_math<EPV>(c, alpha, g, w, mm, vv);
      if (c.optim != SGD) {
#pragma unroll
        for (int i = 0; i < EPV; i += 4) {
          *reinterpret_cast<float4*>(mp + i) = make_float4(mm[i], mm[i + 1], mm[i + 2], mm[i + 3]);
          if (c.optim == ADAM)
            *reinterpret_cast<float4*>(vp + i) = make_float4(vv[i], vv[i + 1], vv[i + 2], vv[i + 3]);
        }
      }
      st16(wp, Vec<DT>::pack(w));
    }
  }
  if (part == 0 && c.N > 1) {
    // the LAST CTA to finish announces prior_done(t) (and, outside SPLIT,
    // def_done(t): there is no second part) to every owner: the next forward's
    // gate then only waits, and the flag leaves as soon as the update is
    // complete instead of after the next gate kernel's own dependency wait
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(c.merge_cnt + p, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
      c.merge_cnt[p] = 0;
      publish2(c, EMB_FLAG_OFF(prior_done), t, true, EMB_FLAG_OFF(def_done), t, c.mode != SPLIT);
    }
  }
  EMB_TR_END(part ? 6 : 4, t);
  pdl_trigger();
}

// ------------------------------------------------------------------ launchers
static int grid_for_warps(long long warps, int cap) {
  long long blocks = (warps + BWD_WARPS - 1) / BWD_WARPS;
  if (blocks < 1) blocks = 1;
  if (blocks > cap) blocks = cap;
  return (int)blocks;
}

// pick the V (16-byte chunks per lane) instantiation and launch it with PDL
#define EMB_LAUNCH_V(V_, KERNEL, DT, GRID, SMEM, ...)                                                   \
  ((V_) <= 1   ? launch_pdl(KERNEL<DT, 1>, dim3(GRID), dim3(BWD_THREADS), (SMEM), s, __VA_ARGS__)     \
   : (V_) <= 2 ? launch_pdl(KERNEL<DT, 2>, dim3(GRID), dim3(BWD_THREADS), (SMEM), s, __VA_ARGS__)     \
   : (V_) <= 4 ? launch_pdl(KERNEL<DT, 4>, dim3(GRID), dim3(BWD_THREADS), (SMEM), s, __VA_ARGS__)     \
   : (V_) <= 8 ? launch_pdl(KERNEL<DT, 8>, dim3(GRID), dim3(BWD_THREADS), (SMEM), s, __VA_ARGS__)     \
               : cudaErrorInvalidValue)

template <int DT>
static cudaError_t coal_dispatch(const DevCtx& c, const LaunchCfg& L, const char* y, int p, int gate_flags,
                                 cudaStream_t s) {
  const int V = (c.cpr + 31) / 32;
  const int ga = grid_for_warps(c.max_chunks, L.nsm * L.reduce_per_sm);
  return EMB_LAUNCH_V(V, coal_reduce_kernel, DT, ga, 0, c, y, p, gate_flags);
}

template <int DT>
static cudaError_t apply_dispatch(const DevCtx& c, const LaunchCfg& L, const char* dY, int p, cudaStream_t s) {
  constexpr int EA = EMB_APPLY_EA(Vec<DT>::EPV);
  const int rpb = BWD_THREADS / c.cpr;
  long long grid = ((long long)c.max_tok + (long long)rpb * EA - 1) / ((long long)rpb * EA);
  if (grid > L.nsm * EMB_APPLY_GRID_PER_SM) grid = L.nsm * EMB_APPLY_GRID_PER_SM;
  if (grid < 1) grid = 1;
  return launch_pdl(coal_apply_kernel<DT>, dim3((int)grid), dim3(BWD_THREADS), 0, s, c, dY, p);
}

cudaError_t launch_coal_apply(const DevCtx& c, const LaunchCfg& L, const void* dY, int p, cudaStream_t s) {
  const char* y = static_cast<const char*>(dY);
  return c.dtype == BF16 ? apply_dispatch<BF16>(c, L, y, p, s) : apply_dispatch<F32>(c, L, y, p, s);
}

cudaError_t launch_coal(const DevCtx& c, const LaunchCfg& L, const void* dY, int p, int gate_flags, cudaStream_t s) {
  const char* y = static_cast<const char*>(dY);
  return c.dtype == BF16 ? coal_dispatch<BF16>(c, L, y, p, gate_flags, s) : coal_dispatch<F32>(c, L, y, p, gate_flags, s);
}

cudaError_t launch_defpush(const DevCtx& c, const LaunchCfg& L, int p, cudaStream_t s) {
  const long long work = (long long)c.max_tok * c.cpr;  // upper bound; counts live on the device
  int grid = (int)((work + BWD_THREADS * 4 - 1) / (BWD_THREADS * 4));
  if (grid < 1) grid = 1;
  if (grid > L.nsm * 2) grid = L.nsm * 2;
  return launch_pdl(defpush_kernel, dim3(grid), dim3(BWD_THREADS), 0, s, c, p);
}

cudaError_t launch_rawpush(const DevCtx& c, const LaunchCfg& L, const void* dY, int n, int p, cudaStream_t s) {
  const long long work = (long long)n * c.cpr;
  int grid = (int)((work + BWD_THREADS * 4 - 1) / (BWD_THREADS * 4));
  if (grid < 1) grid = 1;
  if (grid > L.nsm * 2) grid = L.nsm * 2;
  return launch_pdl(rawpush_kernel, dim3(grid), dim3(BWD_THREADS), 0, s, c, static_cast<const char*>(dY), n, p);
}

template <int DT>
static cudaError_t rawcoal_dispatch(const DevCtx& c, const LaunchCfg& L, int p, cudaStream_t s) {
  const int V = (c.cps + 31) / 32;
  const int ga = grid_for_warps((long long)c.N * c.max_chunks, L.nsm * 4);
  cudaError_t e = EMB_LAUNCH_V(V, rawcoal_a_kernel, DT, ga, 0, c, p);
  if (e != cudaSuccess) return e;
  const size_t smem = (size_t)BWD_WARPS * c.d * 4;
  int gb = c.N * c.max_long;
  if (gb < 1) gb = 1;
  return EMB_LAUNCH_V(V, rawcoal_b_kernel, DT, gb, smem, c, p);
}

cudaError_t launch_rawcoal(const DevCtx& c, const LaunchCfg& L, int p, cudaStream_t s) {
  return c.dtype == BF16 ? rawcoal_dispatch<BF16>(c, L, p, s) : rawcoal_dispatch<F32>(c, L, p, s);
}

cudaError_t launch_merge(const DevCtx& c, const LaunchCfg& L, int p, int part, cudaStream_t s) {
  int G = 1;
  while (G * 2 <= 32 && G * 2 <= c.cps) G *= 2;
  const long long items = (long long)c.N * c.max_tok;  // upper bound
  long long threads = items * G;
  int grid = (int)((threads + BWD_THREADS - 1) / BWD_THREADS);
  if (grid < 1) grid = 1;
  if (grid > L.nsm * 4) grid = L.nsm * 4;  // waits inside: bounded
  const bool raw = (c.mode == RAW);
  const dim3 g(grid), b(BWD_THREADS);
  if (c.dtype == BF16)
    return raw ? launch_pdl(merge_kernel<BF16, true>, g, b, 0, s, c, p, part, G)
               : launch_pdl(merge_kernel<BF16, false>, g, b, 0, s, c, p, part, G);
  return raw ? launch_pdl(merge_kernel<F32, true>, g, b, 0, s, c, p, part, G)
             : launch_pdl(merge_kernel<F32, false>, g, b, 0, s, c, p, part, G);
}

template <int DT>
static cudaError_t preload_dt() {
  const void* fs[] = {(const void*)coal_reduce_kernel<DT, 1>, (const void*)coal_reduce_kernel<DT, 2>,
                      (const void*)coal_reduce_kernel<DT, 4>, (const void*)coal_reduce_kernel<DT, 8>,
                      (const void*)rawcoal_a_kernel<DT, 1>,   (const void*)rawcoal_a_kernel<DT, 2>,
                      (const void*)rawcoal_a_kernel<DT, 4>,   (const void*)rawcoal_a_kernel<DT, 8>,
                      (const void*)rawcoal_b_kernel<DT, 1>,   (const void*)rawcoal_b_kernel<DT, 2>,
                      (const void*)rawcoal_b_kernel<DT, 4>,   (const void*)rawcoal_b_kernel<DT, 8>,
                      (const void*)coal_apply_kernel<DT>,     (const void*)merge_kernel<DT, true>,
                      (const void*)merge_kernel<DT, false>};
  for (const void* f : fs)
    if (cudaError_t e = preload(f)) return e;
  return cudaSuccess;
}

cudaError_t preload_bwd() {
  if (cudaError_t e = preload_dt<F32>()) return e;
  if (cudaError_t e = preload_dt<BF16>()) return e;
  if (cudaError_t e = preload((const void*)defpush_kernel)) return e;
  return preload((const void*)rawpush_kernel);
}

}  // namespace emb
