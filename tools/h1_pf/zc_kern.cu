// SM-driven host-link copies for the h1_pf pump (DMA_PULL / DMA_PUSH):
// pull = zero-copy loads of mapped pinned memory into HBM (H2D direction),
// push = stores from HBM into mapped pinned memory (D2H direction).  SMs keep
// far more reads in flight than a copy engine; does that win the DMA a bigger
// share of a host DRAM the H1 team saturates?
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(1024) k_pull(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t units) {
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (size_t)gridDim.x * blockDim.x;
  size_t u = tid;
  for (; u + 7 * nthr < units; u += 8 * nthr) {
    uint4 r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = __ldcv(src + u + k * nthr);
#pragma unroll
    for (int k = 0; k < 8; ++k) dst[u + k * nthr] = r[k];
  }
  for (; u < units; u += nthr) dst[u] = __ldcv(src + u);
}
__global__ void __launch_bounds__(1024) k_push(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t units) {
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (size_t)gridDim.x * blockDim.x;
  for (size_t u = tid; u < units; u += nthr) dst[u] = __ldcs(src + u);
}
extern "C" int zc_copy(int push, const void* src, void* dst, size_t bytes, int ctas, cudaStream_t st) {
  if (push) k_push<<<ctas, 1024, 0, st>>>((const uint4*)src, (uint4*)dst, bytes / 16);
  else k_pull<<<ctas, 1024, 0, st>>>((const uint4*)src, (uint4*)dst, bytes / 16);
  return (int)cudaGetLastError();
}
