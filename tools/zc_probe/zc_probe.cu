// How fast can SMs pull pinned host memory over PCIe (zero-copy loads), and
// how much of that survives while the copy engines run duplex DMA?  Decides
// whether the host lane's staging ring can be served by a kernel (the
// shuttle) without stealing many SMs from K1.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a zc_probe.cu -o zc_probe
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

template <int UNROLL>
__global__ void pull(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t units) {
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (size_t)gridDim.x * blockDim.x;
  size_t u = tid;
  for (; u + (UNROLL - 1) * nthr < units; u += UNROLL * nthr) {
    uint4 r[UNROLL];
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) r[k] = __ldcv(src + u + k * nthr);
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) dst[u + k * nthr] = r[k];
  }
  for (; u < units; u += nthr) dst[u] = __ldcv(src + u);
}

int main() {
  const size_t bytes = size_t(1) << 30, units = bytes / 16;
  uint4 *h, *hd, *d, *dx, *dy;
  void *hx, *hy;
  cudaHostAlloc((void**)&h, bytes, cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&hd, h, 0);
  cudaMalloc(&d, bytes);
  const size_t db = size_t(256) << 20;
  cudaHostAlloc(&hx, db, 0);
  cudaHostAlloc(&hy, db, 0);
  cudaMalloc(&dx, db);
  cudaMalloc(&dy, db);
  memset(h, 1, bytes);
  cudaStream_t s, s1, s2;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\n");
  for (int dma = 0; dma < 2; ++dma) {
    for (int ctas : {4, 8, 16, 32, 64}) {
      for (int thr : {512, 1024}) {
        for (int unroll : {4, 8}) {
          if (dma)  // keep both copy engines busy for the whole measurement
            for (int k = 0; k < 12; ++k) {
              cudaMemcpyAsync(dx, hx, db, cudaMemcpyHostToDevice, s1);
              cudaMemcpyAsync(hy, dy, db, cudaMemcpyDeviceToHost, s2);
            }
          cudaEventRecord(e0, s);
          if (unroll == 4) pull<4><<<ctas, thr, 0, s>>>(hd, d, units);
          else pull<8><<<ctas, thr, 0, s>>>(hd, d, units);
          cudaEventRecord(e1, s);
          cudaEventSynchronize(e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          cudaDeviceSynchronize();
          printf(" \"%s_ctas%d_thr%d_unroll%d_GBs\": %.2f,\n", dma ? "dma" : "alone", ctas, thr, unroll,
                 bytes / (ms * 1e-3) / 1e9);
        }
      }
    }
  }
  cudaEventRecord(e0, s);
  cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf(" \"copy_engine_h2d_GBs\": %.2f\n}\n", bytes / (ms * 1e-3) / 1e9);
  return 0;
}
