// kernels.cuh — host-callable launchers of the exchange kernels.
#pragma once
#include "common.cuh"

namespace emb {

// done_ctr slots (one per kernel kind that uses the last-block pattern)
enum DoneSlot { K_FWD_IDS = 0, K_IDS = 1, K_COAL = 2, K_DEFPUSH = 3, K_RAWPUSH = 4, K_MERGE0 = 5, K_MERGE1 = 6 };

struct LaunchCfg {
  int nsm;  // SM count of the device
};

// a1-a4: forward (ids all-gather push or prefetch check, wait, pull-gather)
cudaError_t launch_fwd(const DevCtx& c, const LaunchCfg& L, const int* ids, int n, void* out, int p,
                       int prefetched, cudaStream_t s);
// a5: push next ids to every peer, wait, mark D_next (epoch tags)
cudaError_t launch_ids(const DevCtx& c, const LaunchCfg& L, const int* next_ids, int n_next, int p,
                       int do_mark, cudaStream_t s);
// a6 + a8: per-source sort / unique / Alg. 1 split / routing (one CTA per source)
cudaError_t launch_route(const DevCtx& c, const LaunchCfg& L, int p, bool key64, size_t smem, cudaStream_t s);
size_t route_smem_bytes(int max_tok, bool key64);
cudaError_t route_set_smem(bool key64, size_t smem);
// a7 + a9 (+a10 for the prior part): sender coalesce; prior rows pushed to owners, scheduled rows staged
cudaError_t launch_coal(const DevCtx& c, const LaunchCfg& L, const void* dY, int p, cudaStream_t s);
// a12: push the staged scheduled rows to their owners
cudaError_t launch_defpush(const DevCtx& c, const LaunchCfg& L, int p, cudaStream_t s);
// RAW a7/a10: push raw dY column slices; owner-side per-source coalesce
cudaError_t launch_rawpush(const DevCtx& c, const LaunchCfg& L, const void* dY, int n, int p, cudaStream_t s);
cudaError_t launch_rawcoal(const DevCtx& c, const LaunchCfg& L, int p, cudaStream_t s);
// a11 / a12: owner merge (ascending source) + fused sparse optimizer update
cudaError_t launch_merge(const DevCtx& c, const LaunchCfg& L, int p, int part, cudaStream_t s);

}  // namespace emb
