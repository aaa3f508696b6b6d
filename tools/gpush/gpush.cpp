// gpush — can the in-phase grad flush skip host DRAM?  H1 (the shipped loop:
// prefetchw 1 KB ahead, dynamic chunks) on 1e8-param subgroups, its bf16 grads
//   static  read from a host image nobody writes (grads pre-staged: the bound)
//   flush   copied D2H by a copy engine into the host image one subgroup ahead
//           (the engine's in-phase flush today: 2 B DMA write + 2 B H1 read of DRAM)
//   push    streamed by a GPU kernel with SM stores into a ring of R chunk slots
//           (C elements each) that the team consumes chunk by chunk; if the
//           ring stays in the LLC, neither the write nor the read reaches DRAM
// each alone and next to duplex pinned DMA (the streamed windows' traffic).
// Usage: gpush <threads> <params/subgroup> <subgroups per window> <dma 0|1> <mode...>
// env: GP_C (chunk elements, 65536), GP_R (ring slots, 32), GP_CTAS (pusher CTAs, 8)
#include <cuda_runtime.h>
#include <immintrin.h>
#include <sys/mman.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unistd.h>
#include <string>
#include <thread>
#include <vector>

#include "../../paper_2410_21316_b200/csrc/dos_internal.h"

namespace base {
#include "../../paper_2410_21316_b200/csrc/dos_host_kern.inc"
}

extern "C" int gpush_launch(const uint16_t* g, int64_t n, int passes, int64_t C, int R, uint16_t* ring_dev,
                            uint32_t* ready_dev, const uint32_t* consumed_dev, uint32_t* abort_dev, int ctas,
                            cudaStream_t st);

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));       \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

static void* big(size_t b) {
  void* q = mmap(nullptr, b, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(q, b, MADV_HUGEPAGE);
  memset(q, 0, b);
  return q;
}

template <class F>
static double par(int T, F f) {
  std::vector<std::thread> th;
  std::atomic<int> go{0}, ready{0};
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      cpu_set_t cs; CPU_ZERO(&cs); CPU_SET(t, &cs); pthread_setaffinity_np(pthread_self(), sizeof(cs), &cs);
      ready++;
      while (!go.load()) {}
      f(t);
    });
  while (ready.load() < T) {}
  auto t0 = std::chrono::steady_clock::now();
  go = 1;
  for (auto& x : th) x.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int main(int argc, char** argv) {
  if (argc < 6) { fprintf(stderr, "usage: gpush threads params passes dma mode...\n"); return 2; }
  const int T = atoi(argv[1]);
  const int64_t n = (int64_t)atof(argv[2]);
  const int P = atoi(argv[3]);
  const bool dma = atoi(argv[4]) != 0;
  const int64_t C = getenv("GP_C") ? atoll(getenv("GP_C")) : 65536;
  const int R = getenv("GP_R") ? atoi(getenv("GP_R")) : 32;
  const int CTAS = getenv("GP_CTAS") ? atoi(getenv("GP_CTAS")) : 8;
  const int64_t pf = 1024;

  float *p = (float*)big(n * 4), *m = (float*)big(n * 4), *v = (float*)big(n * 4), *p0 = (float*)big(n * 4);
  uint16_t *w = (uint16_t*)big(n * 2), *w0 = (uint16_t*)big(n * 2);
  uint16_t* gimg[2] = {(uint16_t*)big(n * 2), (uint16_t*)big(n * 2)};
  for (auto* gi : gimg) CK(cudaHostRegister(gi, n * 2, cudaHostRegisterDefault));
  auto init = [&] {
    par(T, [&](int t) {
      const int64_t lo = n * t / T, hi = n * (t + 1) / T;
      uint32_t x = 12345u + t;
      for (int64_t i = lo; i < hi; ++i) {
        x = x * 1664525u + 1013904223u;
        p[i] = (float)((int)(x >> 8) - (1 << 23)) * 2.4e-9f; m[i] = p[i] * 0.01f; v[i] = 1e-5f + (x >> 24) * 1e-8f;
        gimg[0][i] = gimg[1][i] = (uint16_t)(0x3c00 + (x & 0x7ff)) ^ (uint16_t)((x >> 20) & 0x8000);
        w[i] = 0;
      }
    });
  };
  init();
  uint16_t* dev_g;
  CK(cudaMalloc(&dev_g, n * 2));
  CK(cudaMemcpy(dev_g, gimg[0], n * 2, cudaMemcpyHostToDevice));
  // ring + flags (mapped pinned)
  uint16_t* ring;
  uint32_t* flags;  // [0,R) ready, [64, 64+R) consumed, [200] abort
  CK(cudaHostAlloc((void**)&ring, (size_t)R * C * 2 + 4096, cudaHostAllocMapped));
  CK(cudaHostAlloc((void**)&flags, 4096, cudaHostAllocMapped));
  uint16_t* ring_dev;
  uint32_t* flags_dev;
  CK(cudaHostGetDevicePointer((void**)&ring_dev, ring, 0));
  CK(cudaHostGetDevicePointer((void**)&flags_dev, flags, 0));
  cudaStream_t fs, ps;
  CK(cudaStreamCreateWithFlags(&fs, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
  cudaEvent_t fev[2];
  for (auto& e : fev) CK(cudaEventCreateWithFlags(&e, cudaEventBlockingSync | cudaEventDisableTiming));
  dos_adam_scalars sc{1e-3f, 0.9f, 0.999f, 1e-8f, 0.1f, 0.001f, 0.f, 0};
  const dos_kscal s = [&] { dos_kscal k{}; k.lr = sc.lr; k.b1 = sc.beta1; k.b2 = sc.beta2; k.eps = sc.eps;
    k.bc1 = sc.bc1; k.bc2 = sc.bc2; k.omb1 = 1.0f - k.b1; k.omb2 = 1.0f - k.b2; k.decay = 1.f; k.adamw = 0; return k; }();

  std::atomic<bool> stop{false};
  std::atomic<uint64_t> moved{0};
  std::thread pump;
  if (dma) {
    const size_t nb = 64u << 20;
    void *hx, *hy, *dx, *dy;
    CK(cudaHostAlloc(&hx, nb, 0)); CK(cudaHostAlloc(&hy, nb, 0)); CK(cudaMalloc(&dx, nb)); CK(cudaMalloc(&dy, nb));
    memset(hx, 1, nb); memset(hy, 2, nb);
    pump = std::thread([=, &stop, &moved] {
      cudaStream_t a, b;
      cudaEvent_t ea, eb;
      cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&ea, cudaEventBlockingSync | cudaEventDisableTiming);
      cudaEventCreateWithFlags(&eb, cudaEventBlockingSync | cudaEventDisableTiming);
      while (!stop.load()) {
        cudaMemcpyAsync(dx, hx, nb, cudaMemcpyHostToDevice, a);
        cudaMemcpyAsync(hy, dy, nb, cudaMemcpyDeviceToHost, b);
        cudaEventRecord(ea, a); cudaEventRecord(eb, b);
        cudaEventSynchronize(ea); cudaEventSynchronize(eb);
        moved += 2 * nb;
      }
    });
    std::this_thread::sleep_for(std::chrono::milliseconds(200));
  }

  bool have_ref = false;
  for (int a = 5; a < argc; ++a) {
    const std::string mode = argv[a];
    for (int rep = 0; rep < 2; ++rep) {  // rep 0: one pass from init (bit check); rep 1: the timed window
      const int passes = rep == 0 ? 1 : P;
      init();
      std::vector<std::atomic<int64_t>> next(passes);
      for (auto& x : next) x = 0;
      const int64_t cpp = (n + C - 1) / C;
      if (mode == "push") {
        memset(flags, 0, 4096);
        CK((cudaError_t)gpush_launch(dev_g, n, passes, C, R, ring_dev, flags_dev, flags_dev + 64, flags_dev + 200,
                                     CTAS, ps));
      }
      if (mode == "flush") {  // the first subgroup's grads before the window (as the engine's flush-ahead)
        CK(cudaMemcpyAsync(gimg[0], dev_g, n * 2, cudaMemcpyDeviceToHost, fs));
        CK(cudaEventRecord(fev[0], fs));
        CK(cudaEventSynchronize(fev[0]));
      }
      std::atomic<int> arrived{0};
      const uint64_t m0 = moved.load();
      const double secs = par(T, [&](int t) {
        for (int i = 0; i < passes; ++i) {
          if (mode == "flush" && t == 0) {
            if (i + 1 < passes) {  // next subgroup's grads D2H while this one updates
              CK(cudaMemcpyAsync(gimg[(i + 1) & 1], dev_g, n * 2, cudaMemcpyDeviceToHost, fs));
              CK(cudaEventRecord(fev[(i + 1) & 1], fs));
            }
          }
          if (mode == "push") {
            volatile uint32_t* ready = flags;
            uint32_t* consumed = flags + 64;
            for (int64_t c; (c = next[i].fetch_add(C)) < n;) {
              const int64_t k = (int64_t)i * cpp + c / C;
              const int slot = (int)(k % R);
              for (uint64_t spins = 0; ready[slot] != (uint32_t)(k + 1); ++spins) {
                _mm_pause();
                if (spins > (1ull << 34)) { fprintf(stderr, "ring stalled at chunk %lld\n", (long long)k); _exit(3); }
              }
              std::atomic_thread_fence(std::memory_order_acquire);
              base::adam_range_pf(p, m, v, ring + (int64_t)slot * C - c, DOS_BF16, w, DOS_BF16, c,
                                  std::min(n, c + C), s, pf);
              __atomic_store_n(&consumed[slot], (uint32_t)(k + 1), __ATOMIC_RELEASE);
            }
          } else {
            const uint16_t* g = mode == "flush" ? gimg[i & 1] : gimg[0];
            for (int64_t c; (c = next[i].fetch_add(1 << 18)) < n;)
              base::adam_range_pf(p, m, v, g, DOS_BF16, w, DOS_BF16, c, std::min<int64_t>(n, c + (1 << 18)), s, pf);
          }
          arrived.fetch_add(1);
          while (arrived.load() < (2 * i + 1) * T) _mm_pause();
          if (mode == "flush" && t == 0 && i + 1 < passes) CK(cudaEventSynchronize(fev[(i + 1) & 1]));
          arrived.fetch_add(1);  // second barrier: nobody starts pass i+1 before its grads landed
          while (arrived.load() < (2 * i + 2) * T) _mm_pause();
        }
      });
      if (mode == "push") CK(cudaStreamSynchronize(ps));
      const double dma_gbs = (moved.load() - m0) / secs / 1e9;
      if (rep == 0) {
        if (!have_ref) { memcpy(p0, p, n * 4); memcpy(w0, w, n * 2); have_ref = true; }
        const bool same = !memcmp(p0, p, n * 4) && !memcmp(w0, w, n * 2);
        if (!same) printf("{\"mode\": \"%s\", \"error\": \"not bit-exact vs the first mode\"}\n", mode.c_str());
        continue;
      }
      printf("{\"mode\": \"%s\", \"threads\": %d, \"dma\": %d, \"C\": %lld, \"R\": %d, \"ctas\": %d, "
             "\"h1_Gparams_s\": %.3f, \"dma_GBs\": %.1f, \"subgroups\": %d, \"secs\": %.3f}\n",
             mode.c_str(), T, dma, (long long)C, R, CTAS, (double)n * passes / secs / 1e9, dma_gbs, passes, secs);
      fflush(stdout);
    }
  }
  stop = true;
  if (pump.joinable()) pump.join();
  return 0;
}
