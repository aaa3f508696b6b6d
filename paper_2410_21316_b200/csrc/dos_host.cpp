// dos_host.cpp — host side of libdos: error reporting, the host thread team,
// H1 entry points (bit-exact host Adam + conversions) and the pinned pool.
//
// H1 replaces the reference's CPU-lane work:
//   CPU_UPDATE   -> adam_step_subgroup (pkg/src/optistate/executor.py:77-100)
//                   = upscale (core.py:201-205) + adam_step_arrays (kernels.py:107-139)
//   CPU_DOWNSCALE-> downscale_rne per batch member (executor.py:228-231)
// The reference runs these single-threaded under the GIL (numba @njit without
// parallel/nogil, kernels.py:90); here a team of pinned threads splits each
// subgroup into contiguous, cache-line aligned chunks.
#include <errno.h>
#include <sched.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <map>
#include <memory>
#include <unordered_map>
#include <vector>

#include "dos_internal.h"

// ---------------------------------------------------------------- errors
static thread_local std::string g_err;

int dos_set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

extern "C" const char* dos_last_error(void) { return g_err.c_str(); }
extern "C" int dos_version(void) { return 1; }

// ---------------------------------------------------------------- ISA pick
static const dos_hk_table& hk() {
  static const dos_hk_table* t = [] {
    __builtin_cpu_init();
    if (__builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
        __builtin_cpu_supports("avx512vl") && __builtin_cpu_supports("avx512dq"))
      return &dos_hk_avx512;
    if (__builtin_cpu_supports("avx2")) return &dos_hk_avx2;
    return &dos_hk_generic;
  }();
  return *t;
}

// ---------------------------------------------------------------- team
// Fork-join pool: thread 0 is the caller; workers 1..n-1 are pinned to the
// process's allowed CPUs (one per core) and sleep between jobs.
namespace {
class Team {
 public:
  explicit Team(int n) : n_(std::max(1, n)) {
    cpu_set_t allowed;
    CPU_ZERO(&allowed);
    std::vector<int> cpus;
    if (sched_getaffinity(0, sizeof allowed, &allowed) == 0)
      for (int c = 0; c < CPU_SETSIZE; ++c)
        if (CPU_ISSET(c, &allowed)) cpus.push_back(c);
    for (int t = 1; t < n_; ++t) {
      threads_.emplace_back([this, t] { loop(t); });
      if (!cpus.empty()) {
        cpu_set_t one;
        CPU_ZERO(&one);
        CPU_SET(cpus[t % cpus.size()], &one);
        pthread_setaffinity_np(threads_.back().native_handle(), sizeof one, &one);
      }
    }
  }
  ~Team() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& th : threads_) th.join();
  }
  int size() const { return n_; }
  // Runs f(t) for t in [0, k) (k <= size) and waits; serialised across callers.
  void run(int k, const std::function<void(int)>& f) {
    std::lock_guard<std::mutex> serial(run_mu_);
    k = std::max(1, std::min(k, n_));
    if (k == 1) {
      f(0);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &f;
      active_ = k;
      pending_ = k - 1;
      ++gen_;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int t) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* job;
      int active;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        job = job_;
        active = active_;
      }
      if (job && t < active) {
        (*job)(t);
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }
  int n_;
  std::vector<std::thread> threads_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int active_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// The team is shared: every parallel section holds a reference for its
// duration, so a resize (dos_set_host_threads) while the engine's host lane or
// a pool commit is inside Team::run only swaps the global pointer; the old
// team is destroyed (its workers joined) when its last user releases it.
std::mutex g_team_mu;
std::shared_ptr<Team> g_team;
int g_team_want = 0;

int default_threads() {
  cpu_set_t allowed;
  CPU_ZERO(&allowed);
  if (sched_getaffinity(0, sizeof allowed, &allowed) == 0) return std::max(1, CPU_COUNT(&allowed));
  return std::max(1, (int)std::thread::hardware_concurrency());
}

std::shared_ptr<Team> team() {
  std::lock_guard<std::mutex> lk(g_team_mu);
  if (!g_team) g_team = std::make_shared<Team>(g_team_want > 0 ? g_team_want : default_threads());
  return g_team;
}

// Splits [0, n) into k chunks aligned to 64 elements (256 B of fp32).
template <class F>
void parallel_chunks(int64_t n, int nthreads, F&& body) {
  const std::shared_ptr<Team> hold = team();  // alive until this section returns
  Team& tm = *hold;
  int k = nthreads > 0 ? std::min(nthreads, tm.size()) : tm.size();
  const int64_t min_chunk = 1 << 16;  // below this, threading costs more than it saves
  k = (int)std::max<int64_t>(1, std::min<int64_t>(k, (n + min_chunk - 1) / min_chunk));
  if (k <= 1) {
    body((int64_t)0, n);
    return;
  }
  const int64_t per = ((n + k - 1) / k + 63) & ~int64_t(63);
  tm.run(k, [&](int t) {
    const int64_t lo = std::min<int64_t>(n, per * t), hi = std::min<int64_t>(n, lo + per);
    if (lo < hi) body(lo, hi);
  });
}

// Splits [0, n) into chunks of `chunk` elements (a multiple of 64) that the
// team's threads claim from a shared counter: a thread that is preempted or
// starved of memory bandwidth (the copy engines share the DRAM) costs the
// section one chunk, not its whole static share.
template <class F>
void parallel_dynamic(int64_t n, int nthreads, int64_t chunk, F&& body) {
  const std::shared_ptr<Team> hold = team();
  Team& tm = *hold;
  int k = nthreads > 0 ? std::min(nthreads, tm.size()) : tm.size();
  k = (int)std::max<int64_t>(1, std::min<int64_t>(k, (n + chunk - 1) / chunk));
  if (k <= 1) {
    body((int64_t)0, n);
    return;
  }
  std::atomic<int64_t> next{0};
  tm.run(k, [&](int) {
    for (int64_t c; (c = next.fetch_add(chunk, std::memory_order_relaxed)) < n;) body(c, std::min(n, c + chunk));
  });
}
}  // namespace

extern "C" int dos_host_threads(void) { return team()->size(); }

extern "C" int dos_set_host_threads(int n) {
  std::lock_guard<std::mutex> lk(g_team_mu);
  g_team_want = n;
  if (g_team && g_team->size() != (n > 0 ? n : default_threads()))
    g_team.reset();  // users still inside a section keep the old team alive
  return DOS_OK;
}

// ---------------------------------------------------------------- H1
// How H1 stores the working copy into a host image: non-temporal 64-byte
// stores (default: no read-for-ownership) or regular cached stores
// (DOS_H1_WSTORE=cached; an A/B knob, profiles/r02_ring_ab.json).
static bool h1_cached_w() {
  static const bool c = [] {
    const char* e = getenv("DOS_H1_WSTORE");
    return e && strcmp(e, "cached") == 0;
  }();
  return c;
}

// DOS_H1_NT=all: p, m, v written back with streaming stores too (A/B knob).
static bool h1_nt_all() {
  static const bool c = [] {
    const char* e = getenv("DOS_H1_NT");
    return e && strcmp(e, "all") == 0;
  }();
  return c;
}

// DOS_H1_PF=<bytes>: write-intent prefetch distance of the default loop
// (0: off).  DOS_H1_CHUNK=<elements>: H1's dynamic chunk (0: one static
// contiguous share per thread).  Defaults from tools/h1_pf on the B200 boxes.
static int64_t env_i64(const char* name, int64_t dflt) {
  const char* e = getenv(name);
  return e && *e ? (int64_t)strtoll(e, nullptr, 10) : dflt;
}
static int64_t h1_pf_bytes() {
  static const int64_t v = std::max<int64_t>(0, env_i64("DOS_H1_PF", 1024));
  return v;
}
static int64_t h1_chunk() {
  static const int64_t v = [] {
    const int64_t c = env_i64("DOS_H1_CHUNK", 1 << 18);
    return c <= 0 ? (int64_t)0 : std::max<int64_t>(64, c & ~int64_t(63));
  }();
  return v;
}

int dos_host_adam(float* p, float* m, float* v, const void* g, int gt, void* lp, int lt, int64_t n,
                  const dos_kscal& s, int nthreads) {
  const dos_hk_table& t = hk();
  if (h1_cached_w() || h1_nt_all()) {
    const auto fn = h1_cached_w() ? t.adam_cached : t.adam_nta;
    parallel_chunks(n, nthreads, [&](int64_t lo, int64_t hi) { fn(p, m, v, g, gt, lp, lt, lo, hi, s); });
    return DOS_OK;
  }
  const int64_t pf = h1_pf_bytes(), chunk = h1_chunk();
  const auto body = [&](int64_t lo, int64_t hi) { t.adam_pf(p, m, v, g, gt, lp, lt, lo, hi, s, pf); };
  if (chunk > 0) parallel_dynamic(n, nthreads, chunk, body);
  else parallel_chunks(n, nthreads, body);
  return DOS_OK;
}

int dos_host_adam_ring(float* p, float* m, float* v, const void* g, int gt, int lt, int64_t n, const dos_kscal& s,
                       int nthreads, const dos_ring& ring, int64_t* last) {
  if (n == 0) return DOS_OK;
  if (lt == DOS_NONE || ring.nslots < 1 || ring.chunk < 64 || !ring.slots || !ring.post || !ring.wait || !last)
    return dos_set_error(DOS_EINVAL, "staging ring: bad configuration");
  const dos_hk_table& t = hk();
  const std::shared_ptr<Team> hold = team();
  Team& tm = *hold;
  int k = nthreads > 0 ? std::min(nthreads, tm.size()) : tm.size();
  k = std::min(k, ring.nthreads);
  const int gsz = gt == DOS_F32 ? 4 : 2;
  // contiguous, 64-element aligned slice per thread (as dos_host_adam)
  const int64_t per = ((n + k - 1) / k + 63) & ~int64_t(63);
  std::atomic<int> err{DOS_OK};
  tm.run(k, [&](int tid) {
    const int64_t lo = std::min<int64_t>(n, per * tid), hi = std::min<int64_t>(n, lo + per);
    int64_t* mine = last + (int64_t)tid * ring.nslots;
    uint16_t* base = ring.slots + (int64_t)tid * ring.nslots * ring.chunk;
    int slot = 0;
    for (int64_t c0 = lo; c0 < hi; c0 += ring.chunk) {
      const int64_t len = std::min(ring.chunk, hi - c0);
      if (mine[slot] >= 0) {  // the slot's previous chunk must have left the host
        const int rc = ring.wait(ring.ctx, mine[slot]);
        if (rc != DOS_OK) {
          err.store(rc);
          return;
        }
        mine[slot] = -1;
      }
      uint16_t* w = base + (int64_t)slot * ring.chunk;
      t.adam_cached(p + c0, m + c0, v + c0, static_cast<const char*>(g) + gsz * c0, gt, w, lt, 0, len, s);
      const int64_t id = ring.post(ring.ctx, w, c0, len);
      if (id < 0) {
        err.store((int)id);
        return;
      }
      mine[slot] = id;
      slot = (slot + 1) % ring.nslots;
    }
  });
  return err.load();
}

int dos_host_adam_gring(float* p, float* m, float* v, int gt, void* lp, int lt, int64_t n, const dos_kscal& s,
                        const dos_gring& r) {
  if (n == 0) return DOS_OK;
  if (gt == DOS_F32 || r.nslots < 1 || r.chunk < 64 || !r.slots || !r.ready || !r.consumed || !r.counts)
    return dos_set_error(DOS_EINVAL, "grad ring: bad configuration");
  const dos_hk_table& t = hk();
  const std::shared_ptr<Team> hold = team();
  Team& tm = *hold;
  const int k = r.nthreads;
  if (k > tm.size()) return dos_set_error(DOS_EINVAL, "grad ring laid out for %d threads, team has %d", k, tm.size());
  const int64_t per = dos_gring_per(n, k), row = (int64_t)k * r.chunk;
  tm.run(k, [&](int tid) {
    const int64_t lo = std::min<int64_t>(n, per * tid), hi = std::min<int64_t>(n, lo + per);
    for (int64_t c = 0; lo + c * r.chunk < hi; ++c) {
      const uint32_t seq = r.seq0 + (uint32_t)c;
      const int slot = (int)(seq % (uint32_t)r.nslots);
      for (int i = 0; (int32_t)(__atomic_load_n(&r.ready[slot], __ATOMIC_ACQUIRE) - (seq + 1)) < 0; ++i) {
        if (i < 1024) __builtin_ia32_pause();
        else std::this_thread::yield();
      }
      const int64_t c0 = lo + c * r.chunk, len = std::min(r.chunk, hi - c0);
      const uint16_t* g = r.slots + (int64_t)slot * row + (int64_t)tid * r.chunk;
      t.adam(p + c0, m + c0, v + c0, g, gt, lp ? static_cast<char*>(lp) + 2 * c0 : nullptr, lp ? lt : DOS_NONE, 0,
             len, s);
      // the last thread done with this row hands its slot back to the copy engine
      if (__atomic_add_fetch(&r.counts[slot], 1, __ATOMIC_ACQ_REL) == dos_gring_row_threads(n, k, r.chunk, c)) {
        __atomic_store_n(&r.counts[slot], 0, __ATOMIC_RELAXED);
        __atomic_store_n(&r.consumed[slot], seq + 1, __ATOMIC_RELEASE);
      }
    }
  });
  return DOS_OK;
}

int dos_host_down(const float* x, void* out, int ot, int64_t n, int nthreads) {
  const dos_hk_table& t = hk();
  parallel_chunks(n, nthreads, [&](int64_t lo, int64_t hi) { t.down(x, out, ot, lo, hi); });
  return DOS_OK;
}

extern "C" int dos_adam_step_host(float* p, float* m, float* v, const void* g, int g_dtype, void* p_lowp,
                                  int lowp_dtype, int64_t n, const dos_adam_scalars* s, int nthreads) {
  if (!s) return dos_set_error(DOS_EINVAL, "scalars must not be NULL");
  if (n < 0) return dos_set_error(DOS_EINVAL, "n must be >= 0");
  if (g_dtype != DOS_F32 && g_dtype != DOS_F16 && g_dtype != DOS_BF16)
    return dos_set_error(DOS_ETYPE, "grad dtype %d unsupported", g_dtype);
  if (lowp_dtype != DOS_NONE && lowp_dtype != DOS_F16 && lowp_dtype != DOS_BF16)
    return dos_set_error(DOS_ETYPE, "working-copy dtype %d unsupported", lowp_dtype);
  if (n == 0) return DOS_OK;
  if (!p || !m || !v || !g || (lowp_dtype != DOS_NONE && !p_lowp)) return dos_set_error(DOS_EINVAL, "NULL buffer");
  return dos_host_adam(p, m, v, g, g_dtype, p_lowp, lowp_dtype, n, dos_make_kscal(s), nthreads);
}

extern "C" int dos_downscale_host(const float* x, void* out, int out_dtype, int64_t n, int nthreads) {
  if (n < 0) return dos_set_error(DOS_EINVAL, "n must be >= 0");
  if (out_dtype != DOS_F16 && out_dtype != DOS_BF16)
    return dos_set_error(DOS_ETYPE, "downscale target dtype %d unsupported", out_dtype);
  if (n == 0) return DOS_OK;
  if (!x || !out) return dos_set_error(DOS_EINVAL, "NULL buffer");
  return dos_host_down(x, out, out_dtype, n, nthreads);
}

extern "C" int dos_upscale_host(const void* x, int in_dtype, float* out, int64_t n, int nthreads) {
  if (n < 0) return dos_set_error(DOS_EINVAL, "n must be >= 0");
  if (in_dtype != DOS_F16 && in_dtype != DOS_BF16)
    return dos_set_error(DOS_ETYPE, "upscale source dtype %d unsupported", in_dtype);
  if (n == 0) return DOS_OK;
  if (!x || !out) return dos_set_error(DOS_EINVAL, "NULL buffer");
  const dos_hk_table& t = hk();
  parallel_chunks(n, nthreads, [&](int64_t lo, int64_t hi) { t.up(x, in_dtype, out, lo, hi); });
  return DOS_OK;
}

// ---------------------------------------------------------------- host memory probe
static volatile uint64_t g_membw_sink;
// The host-DRAM roofline's denominator: one pass of the team over a buffer,
// reading it (mode 0) or copying it (mode 1, glibc memcpy: non-temporal
// stores at these sizes).  Seconds of the pass in *seconds.
extern "C" int dos_host_membw(const void* src, void* dst, size_t bytes, int mode, int nthreads, double* seconds) {
  if (!src || !seconds || (mode == 1 && !dst) || mode < 0 || mode > 1)
    return dos_set_error(DOS_EINVAL, "dos_host_membw: bad arguments");
  const int64_t lines = (int64_t)(bytes / 64);
  std::atomic<uint64_t> sink{0};
  const auto t0 = std::chrono::steady_clock::now();
  parallel_chunks(lines, nthreads, [&](int64_t lo, int64_t hi) {
    const char* s = static_cast<const char*>(src) + lo * 64;
    const size_t n = (size_t)(hi - lo) * 64;
    if (mode == 1) {
      memcpy(static_cast<char*>(dst) + lo * 64, s, n);
      return;
    }
    const uint64_t* q = reinterpret_cast<const uint64_t*>(s);
    uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (size_t i = 0; i + 4 <= n / 8; i += 4) {
      // 1 KB ahead: without it one core keeps too few misses in flight and the
      // pass measures per-core concurrency, not the DRAM (r02: 121 vs ~190 GB/s)
      if ((i & 7) == 0) __builtin_prefetch(q + i + 128, 0, 3);
      a0 ^= q[i];
      a1 ^= q[i + 1];
      a2 ^= q[i + 2];
      a3 ^= q[i + 3];
    }
    sink.fetch_xor(a0 ^ a1 ^ a2 ^ a3, std::memory_order_relaxed);
  });
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  g_membw_sink = sink.load();  // keeps the reads observable
  return DOS_OK;
}

// ---------------------------------------------------------------- pool
// mmap -> MADV_HUGEPAGE -> optional mbind -> parallel first touch by the
// team -> cudaHostRegister.  Registering pre-faulted 2 MB pages is far
// cheaper than cudaHostAlloc's page-by-page pinning of a fresh range.
namespace {
struct Region {
  size_t bytes;
  bool registered;
  bool sparse;                      // dos_host_reserve: committed piecewise
  std::map<size_t, size_t> runs;    // sparse: committed [first, last) 2 MB pages, one registration each
  bool register_cuda;
};
std::mutex g_pool_mu;
std::unordered_map<void*, Region> g_regions;

long sys_mbind(void* addr, unsigned long len, int mode, const unsigned long* nodemask, unsigned long maxnode,
               unsigned flags) {
#ifdef SYS_mbind
  return syscall(SYS_mbind, addr, len, mode, nodemask, maxnode, flags);
#else
  errno = ENOSYS;
  return -1;
#endif
}
}  // namespace

extern "C" int dos_host_alloc(size_t bytes, int numa_node, int register_cuda, void** out) {
  if (!out) return dos_set_error(DOS_EINVAL, "out must not be NULL");
  *out = nullptr;
  if (bytes == 0) bytes = 1;
  const size_t huge = size_t(2) << 20;
  const size_t len = (bytes + huge - 1) & ~(huge - 1);
  void* ptr = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (ptr == MAP_FAILED) return dos_set_error(DOS_ESYS, "mmap(%zu) failed: %s", len, strerror(errno));
  madvise(ptr, len, MADV_HUGEPAGE);
  if (numa_node >= 0 && numa_node < 64) {
    unsigned long mask = 1ul << numa_node;
    if (sys_mbind(ptr, len, 2 /* MPOL_BIND */, &mask, 64, 0) != 0) {
      // not fatal: single-node hosts and containers without CAP_SYS_NICE
    }
  }
  // first touch in parallel, one 2 MB page at a time
  char* base = static_cast<char*>(ptr);
  const int64_t pages = (int64_t)(len / huge);
  parallel_chunks(pages, 0, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) memset(base + i * huge, 0, huge);
  });
  bool registered = false;
  if (register_cuda) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0) {
      const cudaError_t e = cudaHostRegister(ptr, len, cudaHostRegisterDefault);
      if (e != cudaSuccess) {
        munmap(ptr, len);
        return dos_set_error(DOS_ECUDA, "cudaHostRegister(%zu) failed: %s", len, cudaGetErrorString(e));
      }
      registered = true;
    } else {
      cudaGetLastError();  // clear the no-device error; plain memory is still usable
    }
  }
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_regions[ptr] = Region{len, registered, false, {}, false};
  }
  *out = ptr;
  return DOS_OK;
}

// Sparse regions: the address space of a whole flat array is reserved up
// front, but memory is committed (touched, then page-locked and registered)
// only for the ranges that are homed on the host — the subgroups whose fp32
// state lives in HBM never cost host RAM.  Committed runs that touch are
// merged into one registration, so a copy that stays inside a committed run
// is always a pinned DMA.
extern "C" int dos_host_reserve(size_t bytes, int numa_node, int register_cuda, void** out) {
  if (!out) return dos_set_error(DOS_EINVAL, "out must not be NULL");
  *out = nullptr;
  if (bytes == 0) bytes = 1;
  const size_t huge = size_t(2) << 20;
  const size_t len = (bytes + huge - 1) & ~(huge - 1);
  void* ptr = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
  if (ptr == MAP_FAILED) return dos_set_error(DOS_ESYS, "mmap(%zu) failed: %s", len, strerror(errno));
  madvise(ptr, len, MADV_HUGEPAGE);
  if (numa_node >= 0 && numa_node < 64) {
    unsigned long mask = 1ul << numa_node;
    sys_mbind(ptr, len, 2 /* MPOL_BIND */, &mask, 64, 0);  // best effort, as dos_host_alloc
  }
  int ndev = 0;
  const bool reg = register_cuda && cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0;
  if (!reg) cudaGetLastError();
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_regions[ptr] = Region{len, false, true, {}, reg};
  }
  *out = ptr;
  return DOS_OK;
}

extern "C" int dos_host_commit(void* base, size_t offset, size_t len) {
  if (len == 0) return DOS_OK;
  const size_t huge = size_t(2) << 20;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  auto it = g_regions.find(base);
  if (it == g_regions.end()) return dos_set_error(DOS_EINVAL, "pointer %p was not allocated by the host pool", base);
  Region& r = it->second;
  if (!r.sparse) return DOS_OK;  // a dense region is committed whole
  if (offset > r.bytes || len > r.bytes - offset)
    return dos_set_error(DOS_EINVAL, "commit [%zu, +%zu) outside the %zu-byte region", offset, len, r.bytes);
  size_t lo = offset / huge, hi = (offset + len + huge - 1) / huge;
  // runs overlapping or adjacent to [lo, hi) merge into one
  std::vector<std::pair<size_t, size_t>> merged;
  for (auto& kv : r.runs) {
    if (kv.first <= lo && kv.second >= hi) return DOS_OK;  // already committed
    if (kv.second >= lo && kv.first <= hi) merged.push_back(kv);
  }
  size_t nlo = lo, nhi = hi;
  for (auto& kv : merged) {
    nlo = std::min(nlo, kv.first);
    nhi = std::max(nhi, kv.second);
  }
  char* b = static_cast<char*>(base);
  for (auto& kv : merged) {
    if (r.register_cuda) cudaHostUnregister(b + kv.first * huge);
    r.runs.erase(kv.first);
  }
  // first touch of the new pages in parallel (read + write back, so pages that
  // were faulted in earlier keep their contents)
  const int64_t npages4k = (int64_t)((nhi - nlo) * huge / 4096);
  char* start = b + nlo * huge;
  parallel_chunks(npages4k, 0, [&](int64_t a, int64_t e) {
    for (int64_t i = a; i < e; ++i) {
      volatile char* c = start + i * 4096;
      *c = *c;
    }
  });
  if (r.register_cuda) {
    const cudaError_t e = cudaHostRegister(start, (nhi - nlo) * huge, cudaHostRegisterDefault);
    if (e != cudaSuccess) {
      // leave the previously committed runs registered as they were
      for (auto& kv : merged)
        if (cudaHostRegister(b + kv.first * huge, (kv.second - kv.first) * huge, cudaHostRegisterDefault) ==
            cudaSuccess)
          r.runs[kv.first] = kv.second;
      return dos_set_error(DOS_ECUDA, "cudaHostRegister(%zu) failed: %s", (nhi - nlo) * huge,
                           cudaGetErrorString(e));
    }
  }
  r.runs[nlo] = nhi;
  return DOS_OK;
}

extern "C" int64_t dos_host_committed(void* base) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  auto it = g_regions.find(base);
  if (it == g_regions.end()) return dos_set_error(DOS_EINVAL, "pointer %p was not allocated by the host pool", base);
  const Region& r = it->second;
  if (!r.sparse) return (int64_t)r.bytes;
  size_t pages = 0;
  for (auto& kv : r.runs) pages += kv.second - kv.first;
  return (int64_t)(pages * (size_t(2) << 20));
}

extern "C" int dos_host_free(void* ptr) {
  if (!ptr) return DOS_OK;
  Region r;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_regions.find(ptr);
    if (it == g_regions.end()) return dos_set_error(DOS_EINVAL, "pointer %p was not allocated by dos_host_alloc", ptr);
    r = it->second;
    g_regions.erase(it);
  }
  if (r.registered) cudaHostUnregister(ptr);
  if (r.register_cuda)
    for (auto& kv : r.runs) cudaHostUnregister(static_cast<char*>(ptr) + kv.first * (size_t(2) << 20));
  munmap(ptr, r.bytes);
  return DOS_OK;
}
