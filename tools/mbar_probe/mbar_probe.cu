// Minimal mbarrier + cp.async.bulk kernel: does compute-sanitizer's
// synccheck/racecheck model complete_tx?  (evidence for DESIGN.md §4)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void probe(const float* __restrict__ src, float* __restrict__ dst) {
  __shared__ __align__(128) float buf[256];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(1024) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s),
                 "l"(src), "r"(1024), "r"(b)
                 : "memory");
  }
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W_%=;\n}\n" ::"r"(b)
      : "memory");
  dst[threadIdx.x] = buf[threadIdx.x] * 2.0f;
}

int main() {
  float *src, *dst;
  cudaMalloc(&src, 1024);
  cudaMalloc(&dst, 1024);
  float h[256];
  for (int i = 0; i < 256; ++i) h[i] = (float)i;
  cudaMemcpy(src, h, 1024, cudaMemcpyHostToDevice);
  probe<<<1, 256>>>(src, dst);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, dst, 1024, cudaMemcpyDeviceToHost);
  printf("%s %s\n", cudaGetErrorString(e), (h[255] == 510.0f) ? "ok" : "WRONG");
  return 0;
}
