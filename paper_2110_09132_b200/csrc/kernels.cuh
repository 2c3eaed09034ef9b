// kernels.cuh — host-callable launchers of the exchange kernels.
#pragma once
#include "common.cuh"

namespace emb {

struct LaunchCfg {
  int nsm;         // SM count of the device
  int fwd_per_sm;  // forward grid cap, CTAs per SM (env EMB_FWD_GRID_PER_SM, default 4)
  int reduce_per_sm;  // coal_reduce grid cap, CTAs per SM (env EMB_REDUCE_GRID_PER_SM, default 12)
  int fwd_bulk;       // N == 1 forward through the bulk-copy engine (env EMB_FWD_BULK)
};

// Launch with programmatic stream serialization (see pdl_wait / pdl_trigger).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

inline cudaError_t launch_pdl_raw(const void* f, dim3 grid, dim3 block, size_t smem, cudaStream_t s, void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, f, args);
}

// Flag publication protocol: a kernel never
// fences its own stores; the gate that follows it on the same stream (or is
// ordered after it by an event) starts only after the producer completed,
// publishes the producer's flag to every peer (relaxed system-scope stores),
// then waits for the peers' flags.  N == 1 skips the protocol (stream order).
//
// Rows of the backward are addressed by the sender's UNIQUE index i (the
// ascending unique ids of the sort), not by Alg. 1 slot: the split into prior /
// scheduled is an epoch-tagged mark of D_next that every kernel tests per id,
// so no prefix over the split sits on the critical path.  The slot-ordered
// Alg. 1 tables (P_n, D_n) are produced off the critical path (tables).

// Lazy module loading (CUDA 12 default) loads a kernel at its first launch and
// may synchronise the device to do so.  With one-warp gates spinning on flags
// that a not-yet-launched kernel sets, that synchronisation deadlocks until the
// wait bound expires; so every kernel is loaded up front (emb_create).
inline cudaError_t preload(const void* f) {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, f);
}
cudaError_t preload_fwd();
cudaError_t fwd_bulk_set_smem(const DevCtx& c);
cudaError_t preload_bwd();
cudaError_t preload_route();
cudaError_t preload_sort();
cudaError_t preload_gate();

// Peer-flag gates (k_gate.cu): every N > 1 cross-GPU wait runs in a one-warp
// kernel right before the consumer; compute kernels never spin.
enum GateKind {
  GATE_FWD = 0,      // main, before forward(t): prior/def parts of every owner applied
  GATE_SORT = 1,     // aux, before sort(t): every source's ids arrived (+ own merge1(t-2) done)
  GATE_PUB0 = 2,     // before merge(part 0) / rawcoal: every sender's rows arrived
  GATE_PUB1 = 3,     // side, before merge(part 1)
  GATE_SORTED = 4,   // main, before the coalesce: sort(t) done (+ N == 1 prefetch check)
  GATE_MARKED = 5,   // main, before the apply (SPLIT): D_next tags of t+1 done
  GATE_DEFDONE = 6   // side, after merge(part 1): publish def_done(t) to every owner
};
// main / side-stream progress records (device flags, epoch t)
enum SeqIndex { SEQ_BWD = 0, SEQ_APPLIED = 1, SEQ_DEFPUSHED = 2 };
cudaError_t launch_gate(const DevCtx& c, int p, int kind, int flag_arg, cudaStream_t s);

// a1-a4: forward (publish prior_done/def_done of earlier iterations, alpha_t,
// id push or prefetch check, wait for every owner, pull-gather)
cudaError_t launch_fwd(const DevCtx& c, const LaunchCfg& L, const int* ids, int n, void* out, int p,
                       int prefetched, int dedup, cudaStream_t s);
// a6: per-source sort by (dropped, id, position), unique ids, reduce chunks,
// owner routing (slotmap) — auxiliary stream, one iteration ahead
cudaError_t launch_sort(const DevCtx& c, int p, const int* own_ids, int own_n, int from_bwd, bool key64,
                        size_t smem, cudaStream_t s);
size_t sort_smem_bytes(int max_tok, bool key64);
cudaError_t sort_set_smem(int max_tok, bool key64, size_t smem);
// a5: prefetch all-gather of the next ids (markpush) and the D_next epoch tags
// (marktag, + completion flag marked[p]) — Alg. 1 line 4's set
cudaError_t launch_markpush(const DevCtx& c, int p, const int* next_ids, int n_next, int t_mode, cudaStream_t s);
cudaError_t launch_marktag(const DevCtx& c, int p, int do_mark, int set_flag, int t_mode, cudaStream_t s);
// N > 1, after marktag: the owner merge plan of both parts (leaders, sources'
// unique indices), then the completion flag marked[p]
cudaError_t launch_plan(const DevCtx& c, int p, cudaStream_t s);
// a8 presentation: Alg. 1 slot tables P_n ++ D_n, counts p_n (stats / debug; off the critical path)
cudaError_t launch_tables(const DevCtx& c, int p, int t_mode, cudaStream_t s);
// a7 + a9 (+a10 for the prior part): sender coalesce — segmented reduce in
// fp32, long (Zipf-head) segments combined by the last-arriving CTA; N == 1
// applies the optimizer directly, N > 1 pushes prior rows to the owners and
// stages scheduled rows.
cudaError_t launch_coal(const DevCtx& c, const LaunchCfg& L, const void* dY, int p, int gate_flags, cudaStream_t s);
// a7 (multi-chunk combine) + a9/a10 or the N == 1 update: coalesced rows -> owners / stage / shard
cudaError_t launch_coal_apply(const DevCtx& c, const LaunchCfg& L, const void* dY, int p, cudaStream_t s);
// a12: push the staged scheduled rows to their owners (N > 1)
cudaError_t launch_defpush(const DevCtx& c, const LaunchCfg& L, int p, cudaStream_t s);
// RAW a7/a10: push raw dY column slices; owner-side per-source coalesce
cudaError_t launch_rawpush(const DevCtx& c, const LaunchCfg& L, const void* dY, int n, int p, cudaStream_t s);
cudaError_t launch_rawcoal(const DevCtx& c, const LaunchCfg& L, int p, cudaStream_t s);
// a11 / a12: owner merge (ascending source) + fused sparse optimizer update
cudaError_t launch_merge(const DevCtx& c, const LaunchCfg& L, int p, int part, cudaStream_t s);

}  // namespace emb
