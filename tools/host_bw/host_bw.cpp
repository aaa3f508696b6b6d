// host_bw — host DRAM probe: which access pattern reaches the memory's
// bandwidth on these KVM Xeon slices (per-core concurrency vs DRAM).
// Modes (all threads, one contiguous chunk each, 2 MB THP-backed buffers):
//   read64   scalar 64-bit xor (the old dos_host_membw read pass)
//   read512  AVX-512 loads, 4 accumulators
//   readpf   AVX-512 loads + prefetcht0 PF bytes ahead
//   copynt   AVX-512 load + non-temporal store
//   rmw      in-place x = x*a + 1 over 3 streams + 1 read stream + 1 NT write stream (H1's pattern, trivial math)
//   rmwpf    the same with prefetcht0 PF bytes ahead on the 4 read streams
// Usage: host_bw <threads> <MB per buffer> <reps> [PF bytes]
#include <immintrin.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <atomic>

static void* big(size_t b) {
  void* p = mmap(nullptr, b, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(p, b, MADV_HUGEPAGE);
  return p;
}

template <class F>
static double par(int T, F f) {
  std::vector<std::thread> th;
  std::atomic<int> go{0}, ready{0};
  std::chrono::steady_clock::time_point t0;
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      cpu_set_t s; CPU_ZERO(&s); CPU_SET(t, &s); pthread_setaffinity_np(pthread_self(), sizeof(s), &s);
      ready++;
      while (!go.load()) {}
      f(t);
    });
  while (ready.load() < T) {}
  t0 = std::chrono::steady_clock::now();
  go = 1;
  for (auto& x : th) x.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

volatile float sinkf;

int main(int argc, char** argv) {
  int T = atoi(argv[1]);
  size_t MB = atol(argv[2]);
  int reps = atoi(argv[3]);
  long PF = argc > 4 ? atol(argv[4]) : 1024;
  size_t n = MB << 20 >> 2;  // floats per buffer
  float* a = (float*)big(n * 4); float* b = (float*)big(n * 4); float* c = (float*)big(n * 4);
  float* d = (float*)big(n * 4); uint16_t* w = (uint16_t*)big(n * 2); uint16_t* g = (uint16_t*)big(n * 2);
  par(T, [&](int t) { size_t lo = n * t / T, hi = n * (t + 1) / T;
    for (size_t i = lo; i < hi; ++i) { a[i] = 1; b[i] = 2; c[i] = 3; d[i] = 0; w[i] = 0; g[i] = 0x3f80; } });
  auto chunk = [&](int t, size_t& lo, size_t& hi) { lo = (n * t / T) & ~(size_t)15; hi = (n * (t + 1) / T) & ~(size_t)15; };
  const char* names[] = {"read64", "read512", "readpf", "copynt", "rmw", "rmwpf"};
  for (int mode = 0; mode < 6; ++mode) {
    double best = 1e30; double bytes = 0;
    for (int r = 0; r < reps; ++r) {
      double s = par(T, [&](int t) {
        size_t lo, hi; chunk(t, lo, hi);
        if (mode == 0) {
          const uint64_t* q = (const uint64_t*)(a + lo); size_t m = (hi - lo) / 2; uint64_t x0 = 0, x1 = 0, x2 = 0, x3 = 0;
          for (size_t i = 0; i + 4 <= m; i += 4) { x0 ^= q[i]; x1 ^= q[i + 1]; x2 ^= q[i + 2]; x3 ^= q[i + 3]; }
          sinkf = (float)(x0 ^ x1 ^ x2 ^ x3);
        } else if (mode == 1 || mode == 2) {
          __m512 s0 = _mm512_setzero_ps(), s1 = s0, s2 = s0, s3 = s0;
          for (size_t i = lo; i < hi; i += 64) {
            if (mode == 2) { _mm_prefetch((const char*)(a + i) + PF, _MM_HINT_T0); _mm_prefetch((const char*)(a + i) + PF + 64, _MM_HINT_T0);
                             _mm_prefetch((const char*)(a + i) + PF + 128, _MM_HINT_T0); _mm_prefetch((const char*)(a + i) + PF + 192, _MM_HINT_T0); }
            s0 = _mm512_add_ps(s0, _mm512_load_ps(a + i)); s1 = _mm512_add_ps(s1, _mm512_load_ps(a + i + 16));
            s2 = _mm512_add_ps(s2, _mm512_load_ps(a + i + 32)); s3 = _mm512_add_ps(s3, _mm512_load_ps(a + i + 48));
          }
          sinkf = _mm512_reduce_add_ps(_mm512_add_ps(_mm512_add_ps(s0, s1), _mm512_add_ps(s2, s3)));
        } else if (mode == 3) {
          for (size_t i = lo; i < hi; i += 16) _mm512_stream_ps(d + i, _mm512_load_ps(a + i));
        } else {
          const __m512 k = _mm512_set1_ps(0.999f), one = _mm512_set1_ps(1e-7f);
          for (size_t i = lo; i < hi; i += 32) {
            if (mode == 5) {
              _mm_prefetch((const char*)(a + i) + PF, _MM_HINT_T0); _mm_prefetch((const char*)(a + i) + PF + 64, _MM_HINT_T0);
              _mm_prefetch((const char*)(b + i) + PF, _MM_HINT_T0); _mm_prefetch((const char*)(b + i) + PF + 64, _MM_HINT_T0);
              _mm_prefetch((const char*)(c + i) + PF, _MM_HINT_T0); _mm_prefetch((const char*)(c + i) + PF + 64, _MM_HINT_T0);
              _mm_prefetch((const char*)(g + i) + PF / 2, _MM_HINT_T0);
            }
            for (int h = 0; h < 32; h += 16) {
              __m512 gg = _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32(_mm256_load_si256((const __m256i*)(g + i + h))), 16));
              __m512 x = _mm512_add_ps(_mm512_mul_ps(_mm512_load_ps(a + i + h), k), gg);
              __m512 y = _mm512_add_ps(_mm512_mul_ps(_mm512_load_ps(b + i + h), k), one);
              __m512 z = _mm512_add_ps(_mm512_mul_ps(_mm512_load_ps(c + i + h), k), one);
              _mm512_store_ps(a + i + h, x); _mm512_store_ps(b + i + h, y); _mm512_store_ps(c + i + h, z);
              __m256i lw = _mm512_cvtepi32_epi16(_mm512_srli_epi32(_mm512_castps_si512(x), 16));
              if (h == 0) _mm256_stream_si256((__m256i*)(w + i), lw); else _mm256_stream_si256((__m256i*)(w + i + 16), lw);
            }
          }
        }
      });
      best = s < best ? s : best;
    }
    bytes = mode <= 2 ? n * 4.0 : mode == 3 ? n * 8.0 : n * 28.0;
    printf("%-8s T=%d PF=%ld  %.1f GB/s\n", names[mode], T, PF, bytes / best / 1e9);
  }
}
