// p2p_bw.cu — NVLink peer-memory bandwidth of SM-issued loads / stores
// (measurement tool, not the product: SURVEY §8(d) "measure achievable P2P
// store bandwidth"; the denominator for the exchange's forward pull and
// gradient push kernels).  Built and driven by scripts/p2p_bw.py.
//
//   p2p_enable(dev, peer)            cudaDeviceEnablePeerAccess from dev to peer
//   p2p_copy(dev, dst, src, bytes, grid, iters, ms)
//                                    16-byte copies dst <- src by an SM grid on dev
//                                    (src on the peer = pull over NVLink, dst on the
//                                    peer = push), average ms per copy (CUDA events)
//   p2p_copy2(dst0, src0, dst1, src1, bytes, grid, iters, ms0, ms1)
//                                    the same on devices 0 and 1 at once (both
//                                    directions of the link loaded), per-device ms
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void copy16(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n) {
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  // four independent 16-byte loads in flight per thread
  for (; i + 3 * nth < n; i += 4 * nth) {
    const uint4 a = src[i], b = src[i + nth], c = src[i + 2 * nth], d = src[i + 3 * nth];
    dst[i] = a; dst[i + nth] = b; dst[i + 2 * nth] = c; dst[i + 3 * nth] = d;
  }
  for (; i < n; i += nth) dst[i] = src[i];
}

extern "C" int p2p_enable(int dev, int peer) {
  if (cudaSetDevice(dev) != cudaSuccess) return 1;
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) { cudaGetLastError(); return 0; }
  return e == cudaSuccess ? 0 : 2;
}

static int timed(int dev, void* dst, const void* src, size_t bytes, int grid, int iters, cudaStream_t s,
                 cudaEvent_t a, cudaEvent_t b) {
  const size_t n = bytes / 16;
  for (int w = 0; w < 3; ++w) copy16<<<grid, 256, 0, s>>>((uint4*)dst, (const uint4*)src, n);
  cudaEventRecord(a, s);
  for (int it = 0; it < iters; ++it) copy16<<<grid, 256, 0, s>>>((uint4*)dst, (const uint4*)src, n);
  cudaEventRecord(b, s);
  (void)dev;
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

extern "C" int p2p_copy(int dev, void* dst, const void* src, size_t bytes, int grid, int iters, float* ms) {
  if (cudaSetDevice(dev) != cudaSuccess) return 1;
  cudaStream_t s;
  cudaEvent_t a, b;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int rc = timed(dev, dst, src, bytes, grid, iters, s, a, b);
  if (cudaStreamSynchronize(s) != cudaSuccess) rc = 4;
  float t = 0.f;
  cudaEventElapsedTime(&t, a, b);
  *ms = t / iters;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaStreamDestroy(s);
  return rc;
}

extern "C" int p2p_copy2(void* dst0, const void* src0, void* dst1, const void* src1, size_t bytes, int grid,
                         int iters, float* ms0, float* ms1) {
  cudaStream_t s[2];
  cudaEvent_t a[2], b[2];
  for (int d = 0; d < 2; ++d) {
    cudaSetDevice(d);
    cudaStreamCreateWithFlags(&s[d], cudaStreamNonBlocking);
    cudaEventCreate(&a[d]);
    cudaEventCreate(&b[d]);
  }
  int rc = 0;
  cudaSetDevice(0);
  rc |= timed(0, dst0, src0, bytes, grid, iters, s[0], a[0], b[0]);
  cudaSetDevice(1);
  rc |= timed(1, dst1, src1, bytes, grid, iters, s[1], a[1], b[1]);
  float t[2] = {0.f, 0.f};
  for (int d = 0; d < 2; ++d) {
    cudaSetDevice(d);
    if (cudaStreamSynchronize(s[d]) != cudaSuccess) rc |= 4;
    cudaEventElapsedTime(&t[d], a[d], b[d]);
    cudaEventDestroy(a[d]);
    cudaEventDestroy(b[d]);
    cudaStreamDestroy(s[d]);
  }
  *ms0 = t[0] / iters;
  *ms1 = t[1] / iters;
  return rc;
}
