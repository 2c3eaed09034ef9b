// kernels.cuh — host-callable launchers of the exchange kernels.
#pragma once
#include "common.cuh"

namespace emb {

struct LaunchCfg {
  int nsm;  // SM count of the device
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
// fences its own stores; the NEXT kernel on the same stream (or one ordered
// after it by an event), which starts only after the producer completed,
// publishes the producer's flag to every peer (one thread, one system fence),
// then waits for the peers' flags.  N == 1 skips the protocol (stream order).

// a1-a4: forward (publish prior_done/def_done of earlier iterations, id push or
// prefetch check, wait for every owner, pull-gather)
cudaError_t launch_fwd(const DevCtx& c, const LaunchCfg& L, const int* ids, int n, void* out, int p,
                       int prefetched, cudaStream_t s);
// a6: per-source sort by (dropped, id, position) + unique ids (auxiliary stream)
cudaError_t launch_sort(const DevCtx& c, int p, int fwd_pushed, bool key64, size_t smem, cudaStream_t s);
// a5 + a8: prefetch all-gather of the next ids, D_next bitmap, Alg. 1 split of
// every source's unique ids into prior / scheduled slots, reduce chunks
cudaError_t launch_route(const DevCtx& c, int p, const int* next_ids, int n_next, size_t smem, cudaStream_t s);
size_t sort_smem_bytes(int max_tok, bool key64);
size_t route_smem_bytes(long long vocab);
cudaError_t route_set_smem(int max_tok, bool key64, size_t sort_smem, size_t route_smem);
// a7 + a9 (+a10 for the prior part): sender coalesce.  coal_a: one warp per
// chunk of <= C rows (single-chunk slots emitted directly, others leave fp32
// partials); coal_b: one CTA per multi-chunk slot, fixed-order combine.
cudaError_t launch_coal(const DevCtx& c, const LaunchCfg& L, const void* dY, int p, cudaStream_t s);
// a12: push the staged scheduled rows to their owners (N > 1)
cudaError_t launch_defpush(const DevCtx& c, const LaunchCfg& L, int p, cudaStream_t s);
// RAW a7/a10: push raw dY column slices; owner-side per-source coalesce
cudaError_t launch_rawpush(const DevCtx& c, const LaunchCfg& L, const void* dY, int n, int p, cudaStream_t s);
cudaError_t launch_rawcoal(const DevCtx& c, const LaunchCfg& L, int p, cudaStream_t s);
// a11 / a12: owner merge (ascending source) + fused sparse optimizer update
cudaError_t launch_merge(const DevCtx& c, const LaunchCfg& L, int p, int part, cudaStream_t s);

}  // namespace emb
