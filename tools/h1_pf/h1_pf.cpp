// h1_pf — H1 loop variants on the box's host cores, alone and next to duplex
// pinned DMA (two copy engines streaming 256 MB buffers H2D and D2H):
//   base   the shipped loop (dos_host_kern.inc adam_range, NT working copy)
//   pfD    the same element math with prefetcht0 D bytes ahead on p, m, v, g
//   pwD    prefetchw (read-for-ownership) D bytes ahead on p, m, v; prefetcht0 on g
//   split2 each thread walks two halves of its slice alternately (8 read streams)
//   pwdynD prefetchw D bytes ahead + 256K-element dynamic chunks (the shipped default)
//   dynC   base loop over chunks of C elements handed out by an atomic counter
//          (a late or preempted thread costs one chunk, not its whole slice)
// Rates are taken over a >= 1 s window of back-to-back passes; the DMA bytes
// counted are those the pump completed inside the same window.
// Every variant's results are compared bit-for-bit against base's.
// Usage: h1_pf <threads> <params> <reps> <dma 0|1> <variant ...>
#include <cuda_runtime.h>
#include <immintrin.h>
#include <sys/mman.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../paper_2410_21316_b200/csrc/dos_internal.h"

extern "C" int zc_copy(int push, const void* src, void* dst, size_t bytes, int ctas, cudaStream_t st);

namespace base {
#include "../../paper_2410_21316_b200/csrc/dos_host_kern.inc"
}

template <int MODE>  // 1: prefetcht0, 2: prefetchw on the state streams
static void adam_pf(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                    const uint16_t* __restrict__ g, uint16_t* __restrict__ l, int64_t lo, int64_t hi,
                    const dos_kscal s, int64_t dist) {
  int64_t i = lo;
  alignas(64) uint16_t tmp[32];
  for (; i + 32 <= hi; i += 32) {
    char* pp = reinterpret_cast<char*>(p + i) + dist;
    char* mp = reinterpret_cast<char*>(m + i) + dist;
    char* vp = reinterpret_cast<char*>(v + i) + dist;
    if (MODE == 2) {
      _m_prefetchw(pp); _m_prefetchw(pp + 64); _m_prefetchw(mp); _m_prefetchw(mp + 64);
      _m_prefetchw(vp); _m_prefetchw(vp + 64);
    } else {
      _mm_prefetch(pp, _MM_HINT_T0); _mm_prefetch(pp + 64, _MM_HINT_T0); _mm_prefetch(mp, _MM_HINT_T0);
      _mm_prefetch(mp + 64, _MM_HINT_T0); _mm_prefetch(vp, _MM_HINT_T0); _mm_prefetch(vp + 64, _MM_HINT_T0);
    }
    _mm_prefetch(reinterpret_cast<const char*>(g + i) + dist / 2, _MM_HINT_T0);
    for (int k = 0; k < 32; ++k) {
      float pe = p[i + k], me = m[i + k], ve = v[i + k];
      dos_adam_elem(pe, me, ve, dos_bf16_to_f32(g[i + k]), s);
      p[i + k] = pe; m[i + k] = me; v[i + k] = ve;
      tmp[k] = dos_f32_to_bf16(pe);
    }
    _mm512_stream_si512(reinterpret_cast<__m512i*>(l + i), _mm512_load_si512(tmp));
  }
  for (; i < hi; ++i) {
    float pe = p[i], me = m[i], ve = v[i];
    dos_adam_elem(pe, me, ve, dos_bf16_to_f32(g[i]), s);
    p[i] = pe; m[i] = me; v[i] = ve; l[i] = dos_f32_to_bf16(pe);
  }
  _mm_sfence();
}

static void* big(size_t b) {
  void* q = mmap(nullptr, b, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(q, b, MADV_HUGEPAGE);
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
  if (argc < 6) { fprintf(stderr, "usage: h1_pf threads params reps dma variant...\n"); return 2; }
  const int T = atoi(argv[1]);
  const int64_t n = (int64_t)atof(argv[2]);
  const int reps = atoi(argv[3]);
  const bool dma = atoi(argv[4]) != 0;
  float *p = (float*)big(n * 4), *m = (float*)big(n * 4), *v = (float*)big(n * 4);
  uint16_t *g = (uint16_t*)big(n * 2), *w = (uint16_t*)big(n * 2), *w0 = (uint16_t*)big(n * 2);
  float* p0 = (float*)big(n * 4);
  auto init = [&] {
    par(T, [&](int t) {
      const int64_t lo = n * t / T, hi = n * (t + 1) / T;
      uint32_t x = 12345u + t;
      for (int64_t i = lo; i < hi; ++i) {
        x = x * 1664525u + 1013904223u;
        p[i] = (float)((int)(x >> 8) - (1 << 23)) * 2.4e-9f; m[i] = p[i] * 0.01f; v[i] = 1e-5f + (x >> 24) * 1e-8f;
        g[i] = (uint16_t)(0x3c00 + (x & 0x7ff)) ^ (uint16_t)((x >> 20) & 0x8000);
        w[i] = 0;
      }
    });
  };
  dos_adam_scalars sc{1e-3f, 0.9f, 0.999f, 1e-8f, 0.1f, 0.001f, 0.f, 0};
  const dos_kscal s = [&] { dos_kscal k{}; k.lr = sc.lr; k.b1 = sc.beta1; k.b2 = sc.beta2; k.eps = sc.eps;
    k.bc1 = sc.bc1; k.bc2 = sc.bc2; k.omb1 = 1.0f - k.b1; k.omb2 = 1.0f - k.b2; k.decay = 1.f; k.adamw = 0; return k; }();

  // DMA pump: DMA_H2D / DMA_D2H concurrent streams per direction (default 1
  // each; more streams may land on more copy engines = more reads in flight)
  std::atomic<bool> stop{false};
  std::atomic<uint64_t> moved{0}, moved_h2d{0}, moved_d2h{0};
  std::thread pump;
  const int kh = getenv("DMA_H2D") ? atoi(getenv("DMA_H2D")) : 1;
  const int kd = getenv("DMA_D2H") ? atoi(getenv("DMA_D2H")) : 1;
  // DMA_PULL=<ctas>: the H2D direction by SM zero-copy loads instead of the
  // copy engines; DMA_PUSH=<ctas>: the D2H direction by SM stores
  const int pull = getenv("DMA_PULL") ? atoi(getenv("DMA_PULL")) : 0;
  const int push = getenv("DMA_PUSH") ? atoi(getenv("DMA_PUSH")) : 0;
  if (dma && (pull || push)) {
    const size_t nb = 64u << 20;
    void *hx, *hy, *hxd, *hyd, *dx, *dy;
    cudaHostAlloc(&hx, nb, cudaHostAllocMapped); cudaHostAlloc(&hy, nb, cudaHostAllocMapped);
    cudaHostGetDevicePointer(&hxd, hx, 0); cudaHostGetDevicePointer(&hyd, hy, 0);
    cudaMalloc(&dx, nb); cudaMalloc(&dy, nb);
    memset(hx, 1, nb); memset(hy, 2, nb);
    pump = std::thread([=, &stop, &moved, &moved_h2d, &moved_d2h] {
      cudaStream_t a, b;
      cudaEvent_t ea, eb;
      cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&ea, cudaEventBlockingSync | cudaEventDisableTiming);
      cudaEventCreateWithFlags(&eb, cudaEventBlockingSync | cudaEventDisableTiming);
      while (!stop.load()) {
        if (pull) zc_copy(0, hxd, dx, nb, pull, a);
        else cudaMemcpyAsync(dx, hx, nb, cudaMemcpyHostToDevice, a);
        if (push) zc_copy(1, dy, hyd, nb, push, b);
        else cudaMemcpyAsync(hy, dy, nb, cudaMemcpyDeviceToHost, b);
        cudaEventRecord(ea, a); cudaEventRecord(eb, b);
        cudaEventSynchronize(ea); cudaEventSynchronize(eb);
        moved += 2 * nb; moved_h2d += nb; moved_d2h += nb;
      }
    });
    std::this_thread::sleep_for(std::chrono::milliseconds(200));
  } else if (dma) {
    const size_t nb = 64u << 20;
    std::vector<void*> hs, ds;
    for (int i = 0; i < kh + kd; ++i) {
      void *h, *d;
      cudaHostAlloc(&h, nb, 0); cudaMalloc(&d, nb); memset(h, 1 + i, nb);
      hs.push_back(h); ds.push_back(d);
    }
    pump = std::thread([=, &stop, &moved, &moved_h2d, &moved_d2h] {
      std::vector<cudaStream_t> st(kh + kd);
      std::vector<cudaEvent_t> ev(kh + kd);  // blocking-sync events: the pump sleeps, it does not spin on a core
      for (int i = 0; i < kh + kd; ++i) {
        cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&ev[i], cudaEventBlockingSync | cudaEventDisableTiming);
      }
      while (!stop.load()) {
        for (int i = 0; i < kh + kd; ++i) {
          if (i < kh) cudaMemcpyAsync(ds[i], hs[i], nb, cudaMemcpyHostToDevice, st[i]);
          else cudaMemcpyAsync(hs[i], ds[i], nb, cudaMemcpyDeviceToHost, st[i]);
          cudaEventRecord(ev[i], st[i]);
        }
        for (int i = 0; i < kh + kd; ++i) cudaEventSynchronize(ev[i]);
        moved += (uint64_t)(kh + kd) * nb;
        moved_h2d += (uint64_t)kh * nb;
        moved_d2h += (uint64_t)kd * nb;
      }
    });
    std::this_thread::sleep_for(std::chrono::milliseconds(200));
  }
  bool have_ref = false;
  for (int a = 5; a < argc; ++a) {
    const std::string var = argv[a];
    static std::atomic<int64_t> nexts[4096];
    auto pass = [&](int t, int it) {
      std::atomic<int64_t>& next = nexts[it];
      const int64_t per = ((n + T - 1) / T + 63) & ~int64_t(63);
      const int64_t lo = std::min<int64_t>(n, per * t), hi = std::min<int64_t>(n, lo + per);
      if (var == "idle") {  // no host work: the pump's rates alone
        std::this_thread::sleep_for(std::chrono::milliseconds(50));
      } else if (var == "base") {
        base::adam_range(p, m, v, g, DOS_BF16, w, DOS_BF16, lo, hi, s);
      } else if (var.rfind("pf", 0) == 0) {
        adam_pf<1>(p, m, v, g, w, lo, hi, s, atol(var.c_str() + 2));
      } else if (var.rfind("pw", 0) == 0) {
        adam_pf<2>(p, m, v, g, w, lo, hi, s, atol(var.c_str() + 2));
      } else if (var.rfind("pwdyn", 0) == 0) {  // the shipped default: prefetchw D + 256K chunks
        for (int64_t c; (c = next.fetch_add(1 << 18)) < n;)
          adam_pf<2>(p, m, v, g, w, c, std::min(n, c + (1 << 18)), s, atol(var.c_str() + 5));
      } else if (var.rfind("dyn", 0) == 0) {
        const int64_t C = atol(var.c_str() + 3);
        for (int64_t c; (c = next.fetch_add(C)) < n;)
          base::adam_range(p, m, v, g, DOS_BF16, w, DOS_BF16, c, std::min(n, c + C), s);
      } else if (var == "split2") {
        const int64_t mid = (lo + (hi - lo) / 2) & ~int64_t(63);
        for (int64_t a0 = lo, b0 = mid; a0 < mid || b0 < hi; a0 += 4096, b0 += 4096) {
          if (a0 < mid) base::adam_range(p, m, v, g, DOS_BF16, w, DOS_BF16, a0, std::min(mid, a0 + 4096), s);
          if (b0 < hi) base::adam_range(p, m, v, g, DOS_BF16, w, DOS_BF16, b0, std::min(hi, b0 + 4096), s);
        }
      }
    };
    init();
    nexts[0] = 0;
    double best = par(T, [&](int t) { pass(t, 0); });  // the pass the bit check reads
    const bool have = have_ref;
    if (var == "base" && !have_ref) { memcpy(p0, p, n * 4); memcpy(w0, w, n * 2); have_ref = true; }
    const bool same = have && !memcmp(p0, p, n * 4) && !memcmp(w0, w, n * 2);
    // back-to-back passes inside one parallel region (spin barrier between
    // passes), so the window holds H1 work and nothing else
    const int passes = std::max(2, std::min(4000, (int)(reps * 0.25 / best)));
    for (int i = 0; i < passes; ++i) nexts[i] = 0;
    std::atomic<int> arrived{0};
    const uint64_t m0 = moved.load(), mh0 = moved_h2d.load(), md0 = moved_d2h.load();
    const double tsum = par(T, [&](int t) {
      for (int i = 0; i < passes; ++i) {
        pass(t, i);
        arrived.fetch_add(1);
        while (arrived.load() < (i + 1) * T) _mm_pause();
      }
    });
    const double win = tsum;
    const double dma_gbs = (moved.load() - m0) / win / 1e9;
    const double h2d_gbs = (moved_h2d.load() - mh0) / win / 1e9, d2h_gbs = (moved_d2h.load() - md0) / win / 1e9;
    const double h1_rate = (double)n * passes / tsum;
    printf("{\"variant\": \"%s\", \"threads\": %d, \"dma\": %d, \"h1_Gparams_s\": %.3f, \"h1_best_Gparams_s\": %.3f, "
           "\"h1_GBs\": %.1f, \"dma_GBs\": %.1f, \"h2d_streams\": %d, \"d2h_streams\": %d, \"h2d_GBs\": %.1f, "
           "\"d2h_GBs\": %.1f, \"combined_GBs\": %.1f, \"passes\": %d, \"bitexact_vs_base\": %s}\n",
           var.c_str(), T, dma, h1_rate / 1e9, n / best / 1e9, 28.0 * h1_rate / 1e9, dma_gbs, kh, kd, h2d_gbs, d2h_gbs,
           28.0 * h1_rate / 1e9 * (tsum / win) + dma_gbs, passes, (var == "base" || same) ? "true" : "false");
    fflush(stdout);
  }
  stop = true;
  if (pump.joinable()) pump.join();
}
