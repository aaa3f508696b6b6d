// Host-only probe of H1's chunked staging-ring path: dos_host_adam (working
// copy NT-stored into a big image) vs dos_host_adam_ring with no-op ship /
// wait (regular stores into small per-thread rings, no barrier), on this
// machine's cores.  Separates the ring's compute + barrier cost from the
// per-chunk CUDA API cost of shipping.
//   make -C tools/ring_probe && tools/ring_probe/ring_cpu_probe [n] [chunk per thread] [slots per thread]
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <chrono>
#include <vector>

#include "../../paper_2410_21316_b200/csrc/dos_internal.h"

static std::atomic<int64_t> g_ids{0};
static int64_t post(void*, const uint16_t*, int64_t, int64_t) { return g_ids++; }
static int wait(void*, int64_t) { return DOS_OK; }

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 100000000;
  const int64_t chunk = argc > 2 ? atoll(argv[2]) : (1 << 19);
  const int slots = argc > 3 ? atoi(argv[3]) : 4;
  std::vector<float> p(n, 0.01f), m(n, 0.f), v(n, 1e-5f);
  const int nthr = dos_host_threads();
  std::vector<uint16_t> g(n, 0x3F80), w(n), ring((size_t)nthr * slots * chunk);
  std::vector<int64_t> last((size_t)nthr * slots, -1);
  dos_adam_scalars sc{1e-3f, 0.9f, 0.999f, 1e-8f, 0.1f, 0.001f, 0.f, 0};
  const dos_kscal k = dos_make_kscal(&sc);
  auto timeit = [&](auto fn) {
    fn();
    double best = 1e30;
    for (int r = 0; r < 3; ++r) {
      auto t0 = std::chrono::steady_clock::now();
      fn();
      best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    return n / best / 1e9;
  };
  const double nt = timeit([&] { dos_host_adam(p.data(), m.data(), v.data(), g.data(), DOS_BF16, w.data(), DOS_BF16, n, k, 0); });
  const double now = timeit([&] { dos_host_adam(p.data(), m.data(), v.data(), g.data(), DOS_BF16, nullptr, DOS_NONE, n, k, 0); });
  dos_ring r{ring.data(), nthr, slots, chunk, nullptr, post, wait};
  const double rg = timeit([&] { dos_host_adam_ring(p.data(), m.data(), v.data(), g.data(), DOS_BF16, DOS_BF16, n, k, 0, r, last.data()); });
  printf("{\"n\": %lld, \"chunk\": %lld, \"slots\": %d, \"nt_image_Gps\": %.3f, \"no_w_Gps\": %.3f, \"ring_noop_Gps\": %.3f}\n",
         (long long)n, (long long)chunk, slots, nt, now, rg);
  return 0;
}
