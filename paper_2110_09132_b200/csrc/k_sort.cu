// k_sort.cu — a6 of SURVEY §8(a): per-source sort / unique / reduce chunks /
// owner routing, one thread-block CLUSTER per source.
//
// PAPER.md:380 (§4.2.2): "The calculations require a considerable computing
// resource, and the GPU idle time after BP is a good occasion"; Alg. 1
// line 2 D_u = UNIQUE(D_cur[n]) and COALESCE(G) need, per
// source n, the ascending unique ids and the positions of each id in
// ascending position order (reading R12: canonical summation order).
//
// B200 design (DESIGN.md §5 "sort_unique").  A batch of up to 32768 keys is
// too little work for 148 SMs and too much for one: one SM needed 22 us (LM)
// to 62 us (BERT), enough to bound the whole step from the auxiliary stream.
// Here a cluster of CL = 8 (<= 16384 keys) or 16 (<= 32768 keys, non-portable
// size) CTAs shares one source's keys through distributed shared memory
// (DSMEM):
//   keys   (id' << posbits) | pos with id' = L for dropped tokens (pad when
//          pad_id >= 0, out-of-range ids), so dropped keys sort last; a
//          stable LSD radix sort over the id bits only (8-bit digits: LM 3
//          passes, 32K vocabularies 2) keeps equal ids in position order.
//   pass   every CTA ranks its slice (warp match_any ranking into per-warp
//          digit counters), publishes its 256-bin histogram, reads the other
//          CTAs' histograms over DSMEM to get each digit's global start, and
//          scatters every key straight into the destination CTA's shared
//          memory (global position P -> CTA P / S, slot P % S).
//   heads  kept segment heads are counted per CTA, offset across the cluster
//          over DSMEM, and written as uid / useg / perm / slotmap; then the
//          reduce chunks (C rows) of every unique, the chunk descriptors, and
//          the multi-chunk (Zipf-head) list, again offset over DSMEM.
// Nine cluster barriers per sort (LM), no global atomics, deterministic.
#include <cooperative_groups.h>
#include <stddef.h>
#include <stdlib.h>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace emb {

// Two shapes of the same kernel, 256 threads per CTA: a cluster of 8 CTAs
// (portable size) per source for batches up to 16384 keys, or of 16 CTAs
// (non-portable cluster size, opt-in) up to 32768 keys — the tokens-per-rank
// cap of the exchange.  (A single 1024-thread CTA per source was measured
// slower: profiles/r02_tune/sort_join.txt.)
static constexpr int CL8 = 8;
static constexpr int CL16 = 16;
static constexpr int TH8 = 256;
static constexpr int NB = 256;         // bins of an 8-bit digit
static constexpr int DB = 8;

// Exclusive scan of one int per thread over the CTA (TH threads); *total gets the sum.
template <int TH>
__device__ __forceinline__ int cta_exscan(int v, int* tmp, int* total) {
  constexpr int CS_WARPS = TH / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[w] = x;
  __syncthreads();
  int wsum = 0, all = 0;
#pragma unroll
  for (int i = 0; i < CS_WARPS; ++i) {
    const int ti = tmp[i];
    if (i < w) wsum += ti;
    all += ti;
  }
  *total = all;
  __syncthreads();
  return wsum + x - v;
}

// Sum of `v` over the cluster's CTAs with rank < cr (exclusive) and over all.
template <int CL>
__device__ __forceinline__ void cluster_exsum(cg::cluster_group& cluster, int* slot, int cr, int* before, int* all) {
  int b = 0, a = 0;
#pragma unroll
  for (int q = 0; q < CL; ++q) {
    const int x = *cluster.map_shared_rank(slot, q);
    if (q < cr) b += x;
    a += x;
  }
  *before = b;
  *all = a;
}

#ifndef EMB_SORT_SPREAD
#define EMB_SORT_SPREAD 1
#endif
template <typename K, int EPT, int CL, int CS_THREADS>
__global__ void __launch_bounds__(CS_THREADS) csort_kernel(DevCtx c, int p, const int* own_ids, int own_n,
                                                             int from_bwd) {
  constexpr int CS_WARPS = CS_THREADS / 32;
  EMB_TR_ENTRY();
  pdl_wait();
  if (c.pdl_early) pdl_trigger();  // EMB_PDL_EARLY: let the dependent grid launch now
  cg::cluster_group cluster = cg::this_cluster();
  // from_bwd == 3: an N == 1 prefetched sort whose forward joins its event —
  // no device flag consumer, so its completion count needs no fences
  const bool quiet = from_bwd == 3;
  if (quiet) from_bwd = 2;
  constexpr int SMAX = EPT * CS_THREADS;  // keys per CTA slice (max)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* keyA = reinterpret_cast<K*>(smem_raw);
  K* keyB = keyA + SMAX;
  __shared__ int wh[CS_WARPS][NB];  // per-warp digit counts -> exclusive warp offsets
  __shared__ int ch[NB];            // this CTA's digit totals (read by the cluster)
  __shared__ int gs[NB];            // global start of (digit, this CTA)
  __shared__ int tmp[CS_WARPS];
  __shared__ int xs[6];             // over DSMEM: kept heads, kept tokens, chunks, long, first head; queue
  __shared__ int wk[CS_WARPS];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int cr = (int)cluster.block_rank();
  const int n = blockIdx.x / CL;  // source
  // iteration of the batch: from a backward (batch t+1), one past the sort of
  // t that precedes on this stream — valid even if forward(t) has not run yet
  // (an early fork); from a forward (batch t, not prefetched), after it.
  // (from_bwd == 2, N == 1: the sorts of consecutive batches run on two
  // streams and may overlap; only the completion count is published, the
  // epoch is not needed — no slotmap at N == 1)
  // (from_bwd == 2: tt only labels the kernel trace — the sorts of parity p
  // run in order on one stream, the next is the (count+1)-th: t = 2(count+1) - p)
  const uint32_t tt = from_bwd == 2 ? 2u * (__ldcg(c.sort_count + p) + 1u) - (uint32_t)(p & 1)
                      : from_bwd ? __ldcg(c.sorted + (p ^ 1)) + 1 : c.t_rec[p ^ 1] + 1;
  EMB_TR_BEGIN(1, tt);
  EMB_TR_WAITED(1, tt);
  // N > 1: the gate before this kernel published / waited the ids flags.
  // own_ids (N == 1 prefetch): this rank's batch is read straight from the caller.
  const bool own = own_ids != nullptr && n == c.r;
  const int T = own ? own_n : __ldcg(ntok_of(c, c.r, p, n));
  const int* g = own ? own_ids : gids_of(c, c.r, p, n);
  const int S = (T + CL - 1) / CL;  // slice of each CTA (<= SMAX: T <= max_tok <= CL * SMAX)
  const int lo = cr * S;
  const int cnt = max(0, min(T, lo + S) - lo);
  // keys per warp: the slice spread over all warps (ept <= EPT rounds of 32), so that the
  // per-warp serial work (ranking, heads) is ept rounds, not EPT, when the batch is small
  const int ept = EMB_SORT_SPREAD ? (S + CS_THREADS - 1) / CS_THREADS : EPT;
  const int epw = ept * 32;
  const int posbits = c.posbits, idbits = c.idbits;
  const long long L = c.L;

  // ---- load: key = (id' << posbits) | pos, id' = L for dropped tokens (reading R6)
  unsigned fph = 0;  // N == 1 prefetch fingerprint (see fwd_kernel)
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const int i = tid + e * CS_THREADS;
    if (i < cnt) {
      const int gi = lo + i;
      const int id = __ldcg(g + gi);
      fph += prefetch_hash(id, gi);
      long long idp = id;
      if ((unsigned)id >= (unsigned long long)L) idp = L;               // invalid (the forward flags it)
      else if (c.pad_id >= 0 && (long long)id == c.pad_id) idp = L;     // pad: no gradient
      keyA[i] = (K(idp) << posbits) | K(gi);
    }
  }
  if (own) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) fph += __shfl_xor_sync(0xffffffffu, fph, o);
    if (lane == 0 && fph) atomicAdd(&c.fp[p * 4 + 2], fph);
    if (cr == 0 && tid == 0) atomicAdd(&c.fp[p * 4 + 3], (unsigned)T);
  }
  __syncthreads();
  EMB_TR_AT(1, tt, 4);

  // ---- stable LSD radix over the id bits, 8-bit digits, scatter through DSMEM
  const int top = posbits + idbits;
  for (int sh = posbits; sh < top; sh += DB) {
    const unsigned dmask = (1u << min(DB, top - sh)) - 1u;
#pragma unroll
    for (int j = 0; j < NB / 32; ++j) wh[w][lane + 32 * j] = 0;
    __syncwarp();
    K kk[EPT];
    int dg[EPT], rk[EPT];
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      if (r >= ept) break;
      const int i = w * epw + r * 32 + lane;
      const bool valid = i < cnt;
      const unsigned act = __ballot_sync(0xffffffffu, valid);
      dg[r] = 0;
      if (valid) {
        kk[r] = keyA[i];
        dg[r] = (int)((unsigned)(kk[r] >> sh) & dmask);
        const unsigned peers = __match_any_sync(act, dg[r]);
        const int base = wh[w][dg[r]];
        rk[r] = base + __popc(peers & lt);
        __syncwarp(act);
        if (lane == __ffs(peers) - 1) wh[w][dg[r]] = base + __popc(peers);
        __syncwarp(act);
      }
    }
    __syncthreads();
    if (tid < NB) {  // digit d = tid: exclusive offsets over warps, CTA total
      int run = 0;
#pragma unroll 8
      for (int ww = 0; ww < CS_WARPS; ++ww) {
        const int x = wh[ww][tid];
        wh[ww][tid] = run;
        run += x;
      }
      ch[tid] = run;
    }
    cluster.sync();  // every CTA's ch[] is complete
    {
      int pre = 0, tot = 0, all;
      if (tid < NB) cluster_exsum<CL>(cluster, &ch[tid], cr, &pre, &tot);
      const int ex = cta_exscan<CS_THREADS>(tot, tmp, &all);
      if (tid < NB) gs[tid] = ex + pre;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      if (r >= ept) break;
      const int i = w * epw + r * 32 + lane;
      if (i < cnt) {
        const int P = gs[dg[r]] + wh[w][dg[r]] + rk[r];
        const int dst = P / S;
        *cluster.map_shared_rank(keyB + (P - dst * S), dst) = kk[r];
      }
    }
    cluster.sync();  // scatters landed; nobody reads ch[] / keyA any more
    K* sw = keyA; keyA = keyB; keyB = sw;
  }

  EMB_TR_AT(1, tt, 5);
  // ---- heads -> unique kept ids (ascending), segments, owner routing
  const size_t bpn = pn(c, p, n) * (size_t)c.max_tok;
  int* perm = c.perm + bpn;
  int* uid = c.uid + bpn;
  int* useg = c.useg + pn(c, p, n) * (size_t)(c.max_tok + 1);
  int* hpos = reinterpret_cast<int*>(keyB);  // segment starts of this CTA's uniques (keyB is free now)
  const K posmask = (K(1) << posbits) - 1;
  K prev_last = K(0);
  if (cr > 0 && cnt > 0) prev_last = *cluster.map_shared_rank(keyA + (S - 1), cr - 1);
  if (tid == 0) xs[4] = 0x7fffffff;
  __syncthreads();
  int kept_heads = 0, kept_tok = 0, first_head = 0x7fffffff;
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    if (r >= ept) break;
    const int i = w * epw + r * 32 + lane;
    const bool valid = i < cnt;
    bool head = false, keep = false;
    if (valid) {
      const K key = keyA[i];
      const long long idp = (long long)(key >> posbits);
      keep = idp < L;
      const K prev = (i > 0) ? keyA[i - 1] : prev_last;
      head = keep && ((i == 0 && cr == 0) || (prev >> posbits) != (key >> posbits));
      if (head) first_head = min(first_head, lo + i);
    }
    kept_heads += __popc(__ballot_sync(0xffffffffu, head));
    kept_tok += __popc(__ballot_sync(0xffffffffu, valid && keep));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) first_head = min(first_head, __shfl_xor_sync(0xffffffffu, first_head, o));
  if (lane == 0) {
    wk[w] = kept_heads;
    if (first_head != 0x7fffffff) atomicMin(&xs[4], first_head);
  }
  {
    int tk_all;
    cta_exscan<CS_THREADS>(lane == 0 ? kept_tok : 0, tmp, &tk_all);
    if (tid == 0) xs[1] = tk_all;
  }
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int ww = 0; ww < CS_WARPS; ++ww) { const int x = wk[ww]; wk[ww] = run; run += x; }
    xs[0] = run;
  }
  cluster.sync();  // xs[0] (kept heads), xs[1] (kept tokens), xs[4] (first kept head) of every CTA
  int kb, U, tkb, Tk;
  cluster_exsum<CL>(cluster, &xs[0], cr, &kb, &U);
  cluster_exsum<CL>(cluster, &xs[1], cr, &tkb, &Tk);
  (void)tkb;
  int next_first = Tk;  // end of this CTA's last segment: the next kept head, else the first dropped key
  for (int q = CL - 1; q > cr; --q) {
    const int f = *cluster.map_shared_rank(&xs[4], q);
    if (f != 0x7fffffff) next_first = f;
  }
  {
    int kbase = wk[w];  // local unique index
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      if (r >= ept) break;
      const int i = w * epw + r * 32 + lane;
      const bool valid = i < cnt;
      bool head = false;
      K key = K(0);
      if (valid) {
        key = keyA[i];
        const bool keep = (long long)(key >> posbits) < L;
        const K prev = (i > 0) ? keyA[i - 1] : prev_last;
        head = keep && ((i == 0 && cr == 0) || (prev >> posbits) != (key >> posbits));
      }
      const unsigned hm = __ballot_sync(0xffffffffu, head);
      if (valid) {
        perm[lo + i] = (int)(key & posmask);
        if (head) {
          const int j = kbase + __popc(hm & lt);
          const int k = kb + j;
          const int id = (int)(key >> posbits);
          uid[k] = id;
          useg[k] = lo + i;
          hpos[j] = lo + i;
          if (c.N > 1) c.slotmap[((size_t)p * c.L + id) * c.N + n] = ((unsigned long long)tt << 32) | (unsigned)k;
        }
      }
      kbase += __popc(hm);
    }
  }
  if (cr == 0 && tid == 0) useg[U] = Tk;  // end of the last kept segment (kept keys sort first)
  __syncthreads();  // hpos[] complete

  EMB_TR_AT(1, tt, 6);
  // ---- reduce chunks of C rows per unique: descriptors, multi-chunk list
  //      (segment ends from hpos / next_first: no global round trip)
  int* chunk_off = c.chunk_off + pn(c, p, n) * (size_t)(c.max_tok + 1);
  int4* chunk_desc = c.chunk_desc + pn(c, p, n) * (size_t)c.max_chunks;
  int* long_u = c.long_u + pn(c, p, n) * (size_t)c.max_long;
  int* upos = c.upos + bpn;
  const int hc = xs[0];  // this CTA's uniques: [kb, kb + hc)
  int my_ch = 0, my_long = 0;
  for (int j = tid; j < hc; j += CS_THREADS) {
    const int e = (j + 1 < hc) ? hpos[j + 1] : next_first;
    const int nch = (e - hpos[j] + c.C - 1) / c.C;
    my_ch += nch;
    my_long += nch > 1;
  }
  {
    int a, b;
    cta_exscan<CS_THREADS>(my_ch, tmp, &a);
    cta_exscan<CS_THREADS>(my_long, tmp, &b);
    if (tid == 0) { xs[2] = a; xs[3] = b; xs[5] = 0; }
  }
  cluster.sync();
  int cb, NCH, lb, NLONG;
  cluster_exsum<CL>(cluster, &xs[2], cr, &cb, &NCH);
  cluster_exsum<CL>(cluster, &xs[3], cr, &lb, &NLONG);
  constexpr int QMAX = 32, QMIN = 8;  // uniques of > QMIN chunks: descriptors written by the whole CTA
  __shared__ int4 lq[QMAX];
  __shared__ int lq_off[QMAX];
  for (int j0 = 0; j0 < hc; j0 += CS_THREADS) {
    const int j = j0 + tid;
    const int k = kb + j;
    int a = 0, b = 0, nch = 0;
    if (j < hc) {
      a = hpos[j];
      b = (j + 1 < hc) ? hpos[j + 1] : next_first;
      nch = (b - a + c.C - 1) / c.C;
    }
    int tch, tlong;
    const int och = cta_exscan<CS_THREADS>(nch, tmp, &tch);
    const int olong = cta_exscan<CS_THREADS>(nch > 1 ? 1 : 0, tmp, &tlong);
    if (j < hc) {
      const int off = cb + och;
      chunk_off[k] = off;
      upos[k] = (b - a == 1) ? (int)(keyA[a - lo] & posmask) : -1;  // single-row unique: the apply reads dY there
      int qs = -1;
      if (nch > QMIN) {
        qs = atomicAdd(&xs[5], 1);
        if (qs < QMAX) {
          lq[qs] = make_int4(k, a, b, nch);
          lq_off[qs] = off;
        }
      }
      if (qs < 0 || qs >= QMAX) {
        if (b - a == 1)  // single-row unique: its position (the head key, in this CTA's slice) rides along
          chunk_desc[off] = make_int4(k, a, b, 1 | ((int)(keyA[a - lo] & posmask) + 1) << DESC_POS_SHIFT);
        else
          for (int q = 0; q < nch; ++q) chunk_desc[off + q] = make_int4(k, a + q * c.C, min(b, a + (q + 1) * c.C), nch);
      }
      if (nch > 1) long_u[lb + olong] = k;
    }
    cb += tch;
    lb += tlong;
  }
  __syncthreads();
  for (int e = 0; e < min(xs[5], QMAX); ++e) {  // Zipf-head uniques: descriptors by the whole CTA
    const int4 u = lq[e];
    for (int q = tid; q < u.w; q += CS_THREADS)
      chunk_desc[lq_off[e] + q] = make_int4(u.x, u.y + q * c.C, min(u.z, u.y + (q + 1) * c.C), u.w);
  }
  if (cr == 0 && tid == 0) {
    chunk_off[U] = NCH;
    int* cn = c.counts + pn(c, p, n) * CNT_W;
    cn[CNT_T] = T;
    cn[CNT_U] = U;
    cn[CNT_NCH] = NCH;
    cn[CNT_NLONG] = NLONG;
  }
  EMB_TR_AT(1, tt, 7);
  cluster.sync();  // no CTA exits while a peer may still read its shared memory
  if (quiet) {
    if (cr == 0 && tid == 0) atomicAdd(&c.sort_count[p], 1u);  // trace labels / later GATE_SORTED counts
  } else if (cr == 0 && tid == 0) {
    // sort of parity p complete once every source's cluster arrived: the gate
    // before the coalesce waits for sorted[p] (no host event on the main stream)
    __threadfence();
    if (atomicAdd(&c.sort_cnt[p], 1u) == (unsigned)c.N - 1) {
      c.sort_cnt[p] = 0;
      __threadfence();
      if (from_bwd != 2) st_release_gpu(&c.sorted[p], tt);
      atomicAdd(&c.sort_count[p], 1u);  // after the fence: GATE_SORTED waits the count
    }
  }
  EMB_TR_END(1, tt);
  pdl_trigger();
}

// Shape choice: the 8-CTA cluster up to 8 x 2048 keys per source, the 16-CTA
// cluster above (up to 16 x 2048).
static int sort_cl(int max_tok) { return max_tok <= CL8 * 8 * TH8 ? CL8 : CL16; }

static int cs_ept(int max_tok) {
  const int cl = sort_cl(max_tok);
  const int per = (max_tok + cl - 1) / cl;
  const int need = (per + TH8 - 1) / TH8;
  const int opts[] = {1, 2, 3, 4, 6, 8};
  for (int e : opts)
    if (e >= need) return e;
  return -1;
}

size_t sort_smem_bytes(int max_tok, bool key64) {
  const int e = cs_ept(max_tok);
  if (e < 0) return (size_t)1 << 30;
  return (size_t)2 * e * TH8 * (key64 ? 8 : 4);
}

template <typename K, int CL>
static void* csort_fn_shape(int ept) {
  switch (ept) {
    case 1: return (void*)csort_kernel<K, 1, CL, TH8>;
    case 2: return (void*)csort_kernel<K, 2, CL, TH8>;
    case 3: return (void*)csort_kernel<K, 3, CL, TH8>;
    case 4: return (void*)csort_kernel<K, 4, CL, TH8>;
    case 6: return (void*)csort_kernel<K, 6, CL, TH8>;
    case 8: return (void*)csort_kernel<K, 8, CL, TH8>;
    default: return nullptr;
  }
}

template <typename K>
static void* csort_fn(int max_tok) {
  const int e = cs_ept(max_tok);
  return sort_cl(max_tok) == CL8 ? csort_fn_shape<K, CL8>(e) : csort_fn_shape<K, CL16>(e);
}

cudaError_t sort_set_smem(int max_tok, bool key64, size_t smem) {
  void* f = key64 ? csort_fn<unsigned long long>(max_tok) : csort_fn<uint32_t>(max_tok);
  if (!f) return cudaErrorInvalidValue;
  if (sort_cl(max_tok) == CL16) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  if (smem > 48 * 1024) return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return cudaSuccess;
}

cudaError_t launch_sort(const DevCtx& c, int p, const int* own_ids, int own_n, int from_bwd, bool key64,
                        size_t smem, cudaStream_t s) {
  void* f = key64 ? csort_fn<unsigned long long>(c.max_tok) : csort_fn<uint32_t>(c.max_tok);
  if (!f) return cudaErrorInvalidValue;
  const int cl = sort_cl(c.max_tok);
  DevCtx cc = c;
  void* args[] = {&cc, &p, &own_ids, &own_n, &from_bwd};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(c.N * cl);
  cfg.blockDim = dim3(TH8);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelExC(&cfg, f, args);
}

cudaError_t preload_sort() {
  for (int e : {1, 2, 3, 4, 6, 8}) {
    for (void* f : {csort_fn_shape<uint32_t, CL8>(e), csort_fn_shape<unsigned long long, CL8>(e),
                    csort_fn_shape<uint32_t, CL16>(e), csort_fn_shape<unsigned long long, CL16>(e)})
      if (cudaError_t r = preload(f)) return r;
  }
  return cudaSuccess;
}

}  // namespace emb
