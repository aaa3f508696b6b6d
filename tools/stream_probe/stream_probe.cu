// Is K1's sensitivity to concurrent host-link DMA a property of its access
// pattern (five separate HBM streams: p, m, v, g in; p, m, v, w out) rather
// than of its pipeline?  Two register-path kernels with K1's exact byte
// pattern (28 B/element) and trivial math:
//   split:       p, m, v as three separate fp32 arrays (K1's layout today)
//   interleaved: p, m, v tile-interleaved in one array (4096-element tiles)
// each timed alone and while duplex pinned DMA runs on two other streams.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a stream_probe.cu -o stream_probe
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <atomic>
#include <thread>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));           \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

constexpr int TE = 4096;  // tile elements (as K1)

__device__ __forceinline__ float4 upd(float4 a, float4 b, float4 c, float g) {
  return make_float4(a.x + b.x * g + c.x, a.y + b.y * g + c.y, a.z + b.z * g + c.z, a.w + b.w * g + c.w);
}

__global__ void k_split(float4* p, float4* m, float4* v, const uint2* g, uint2* w, long n4) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    float4 a = __ldcs(p + i), b = __ldcs(m + i), c = __ldcs(v + i);
    uint2 gg = __ldcs(g + i);
    float gf = __uint_as_float(gg.x << 16);
    float4 na = upd(a, b, c, gf), nb = upd(b, c, a, gf), nc = upd(c, a, b, gf);
    __stcs(p + i, na);
    __stcs(m + i, nb);
    __stcs(v + i, nc);
    __stcs(w + i, make_uint2(__float_as_uint(na.x) >> 16, __float_as_uint(na.y) >> 16));
  }
}

// s: per tile [p(TE) | m(TE) | v(TE)] fp32
__global__ void k_inter(float4* s, const uint2* g, uint2* w, long n4) {
  constexpr long T4 = TE / 4;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    const long t = i / T4, o = i % T4;
    float4* base = s + t * 3 * T4 + o;
    float4 a = __ldcs(base), b = __ldcs(base + T4), c = __ldcs(base + 2 * T4);
    uint2 gg = __ldcs(g + i);
    float gf = __uint_as_float(gg.x << 16);
    float4 na = upd(a, b, c, gf), nb = upd(b, c, a, gf), nc = upd(c, a, b, gf);
    __stcs(base, na);
    __stcs(base + T4, nb);
    __stcs(base + 2 * T4, nc);
    __stcs(w + i, make_uint2(__float_as_uint(na.x) >> 16, __float_as_uint(na.y) >> 16));
  }
}

int main() {
  const long n = 100000000L - 100000000L % TE;
  const long n4 = n / 4;
  float *p, *m, *v, *s;
  uint2 *g, *w;
  CK(cudaMalloc(&p, n * 4));
  CK(cudaMalloc(&m, n * 4));
  CK(cudaMalloc(&v, n * 4));
  CK(cudaMalloc(&s, n * 12));
  CK(cudaMalloc(&g, n * 2));
  CK(cudaMalloc(&w, n * 2));
  CK(cudaMemset(p, 0, n * 4));
  CK(cudaMemset(m, 0, n * 4));
  CK(cudaMemset(v, 0, n * 4));
  CK(cudaMemset(s, 0, n * 12));
  CK(cudaMemset(g, 0, n * 2));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int grid = sms * 4, block = 512;
  const size_t nb = 256ul << 20;
  void *hx, *hy, *dx, *dy;
  CK(cudaMallocHost(&hx, nb));
  CK(cudaMallocHost(&hy, nb));
  CK(cudaMalloc(&dx, nb));
  CK(cudaMalloc(&dy, nb));
  cudaStream_t ks, s1, s2;
  CK(cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  std::atomic<bool> stop{false}, dma{false};
  std::thread pump([&] {
    CK(cudaSetDevice(0));
    while (!stop) {
      if (!dma) {
        std::this_thread::yield();
        continue;
      }
      CK(cudaMemcpyAsync(dx, hx, nb, cudaMemcpyHostToDevice, s1));
      CK(cudaMemcpyAsync(hy, dy, nb, cudaMemcpyDeviceToHost, s2));
      CK(cudaStreamSynchronize(s1));
      CK(cudaStreamSynchronize(s2));
    }
  });
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](int which) {
    const int reps = 20;
    for (int r = 0; r < 2; ++r) {
      if (which == 0) k_split<<<grid, block, 0, ks>>>((float4*)p, (float4*)m, (float4*)v, g, w, n4);
      else k_inter<<<grid, block, 0, ks>>>((float4*)s, g, w, n4);
    }
    CK(cudaEventRecord(e0, ks));
    for (int r = 0; r < reps; ++r) {
      if (which == 0) k_split<<<grid, block, 0, ks>>>((float4*)p, (float4*)m, (float4*)v, g, w, n4);
      else k_inter<<<grid, block, 0, ks>>>((float4*)s, g, w, n4);
    }
    CK(cudaEventRecord(e1, ks));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return 28.0 * n * reps / (ms * 1e-3) / 1e9;
  };
  for (int round = 0; round < 2; ++round) {
    for (int which = 0; which < 2; ++which) {
      dma = false;
      std::this_thread::sleep_for(std::chrono::milliseconds(50));
      const double alone = timeit(which);
      dma = true;
      std::this_thread::sleep_for(std::chrono::milliseconds(100));
      const double busy = timeit(which);
      printf("{\"kernel\": \"%s\", \"alone_GBs\": %.1f, \"duplex_dma_GBs\": %.1f, \"loss\": %.4f}\n",
             which == 0 ? "split" : "interleaved", alone, busy, 1.0 - busy / alone);
      fflush(stdout);
    }
  }
  stop = true;
  dma = false;
  pump.join();
  return 0;
}
