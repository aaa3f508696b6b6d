// Grad pusher: a persistent kernel that streams a subgroup's bf16 grads from
// HBM into a small ring of pinned host slots with SM stores (posted PCIe
// writes, no copy engine), chunk k into slot k % R once the host team has
// consumed chunk k - R, then publishes ready[slot] = k + 1.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(512) k_gpush(const uint16_t* g, int64_t n, int passes, int64_t C, int R,
                                               uint16_t* ring, uint32_t* ready, const uint32_t* consumed,
                                               uint32_t* abort_flag) {
  const int64_t cpp = (n + C - 1) / C;
  const int64_t K = cpp * passes;
  __shared__ int s_quit;
  for (int64_t k = blockIdx.x; k < K; k += gridDim.x) {
    const int slot = (int)(k % R);
    if (threadIdx.x == 0) {
      s_quit = 0;
      if (k >= R) {
        const uint64_t t0 = gtime();
        while (ld_acquire_sys(&consumed[slot]) < (uint32_t)(k - R + 1)) {
          if (ld_acquire_sys(abort_flag) || gtime() - t0 > 20ull * 1000000000ull) {
            s_quit = 1;
            break;
          }
          __nanosleep(256);
        }
      }
    }
    __syncthreads();
    if (s_quit) return;
    const int64_t c = (k % cpp) * C;
    const int64_t len = n - c < C ? n - c : C;
    const uint4* src = reinterpret_cast<const uint4*>(g + c);
    uint4* dst = reinterpret_cast<uint4*>(ring + (int64_t)slot * C);
    const int64_t units = len * 2 / 16;
    for (int64_t u = threadIdx.x; u < units; u += blockDim.x) dst[u] = __ldcs(src + u);
    for (int64_t e = units * 8 + threadIdx.x; e < len; e += blockDim.x) ring[(int64_t)slot * C + e] = g[c + e];
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      st_release_sys(&ready[slot], (uint32_t)(k + 1));
    }
  }
}
}  // namespace

extern "C" int gpush_launch(const uint16_t* g, int64_t n, int passes, int64_t C, int R, uint16_t* ring_dev,
                            uint32_t* ready_dev, const uint32_t* consumed_dev, uint32_t* abort_dev, int ctas,
                            cudaStream_t st) {
  k_gpush<<<ctas, 512, 0, st>>>(g, n, passes, C, R, ring_dev, ready_dev, consumed_dev, abort_dev);
  return (int)cudaGetLastError();
}
