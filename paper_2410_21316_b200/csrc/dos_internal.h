// dos_internal.h — declarations shared by the libdos translation units.
#pragma once
#include <stdint.h>

#include "../../include/dos.h"
#include "dos_numerics.h"

#ifdef __CUDACC__
#include <cuda_runtime.h>
#else
#include <cuda_runtime_api.h>
#endif

// Records a thread-local message (printf format) and returns `code`.
int dos_set_error(int code, const char* fmt, ...);

// Per-launch scalars from the C-ABI struct (fp32 arithmetic on the host).
dos_kscal dos_make_kscal(const dos_adam_scalars* s);

// Peer destinations of the working copy (fused all-gather); element 0 of
// each pointer corresponds to element 0 of the launch's range.
struct dos_peers {
  int n;
  uint16_t* p[DOS_MAX_PEERS];
};
dos_peers dos_peers_offset(const dos_peers& pr, int64_t elems);

// Sources of the fused reduce-scatter: p[r] is where the launch's range
// starts in rank r's full-model grad buffer (16-bit, r = 0..n-1 in rank
// order; p[self] is the local buffer).  The grad a kernel uses is
// lowp(((w0 + w1) + w2) + ...) with fp32 RN adds in rank order, then
// lowp(widen(that) * scale) if scale != 1 (ZeRO-3 averaging).  n == 0: off.
struct dos_gsrc {
  int n;
  int self;
  float scale;
  const uint16_t* p[DOS_MAX_PEERS + 1];
};
dos_gsrc dos_gsrc_offset(const dos_gsrc& gs, int64_t elems);

// K1 launch without argument validation (used by the engine).  With
// gs.n > 0 the grads are the reduce-scatter of gs (g must be gs.p[gs.self]).
int dos_adam_launch(float* p, float* m, float* v, const void* g, int gt, void* lp, int lt, int64_t n,
                    const dos_kscal& s, cudaStream_t st, const dos_peers& pr = dos_peers{0, {}},
                    const dos_gsrc& gs = dos_gsrc{0, 0, 1.0f, {}});
// Stand-alone reduce-scatter of a range: out = the reduced grads of gs (n elements).
int dos_reduce_launch(void* out, int dt, int64_t n, const dos_gsrc& gs, cudaStream_t st);

// Host kernels (dos_host.cpp); the calling thread joins the team.
int dos_host_adam(float* p, float* m, float* v, const void* g, int gt, void* lp, int lt, int64_t n,
                  const dos_kscal& s, int nthreads);
int dos_host_down(const float* x, void* out, int ot, int64_t n, int nthreads);

// One ISA variant of the host loops (dos_host_isa.cpp, built per ISA).
struct dos_hk_table {
  void (*adam)(float*, float*, float*, const void*, int, void*, int, int64_t, int64_t, const dos_kscal&);
  void (*down)(const float*, void*, int, int64_t, int64_t);
  void (*up)(const void*, int, float*, int64_t, int64_t);
  void (*adam_cached)(float*, float*, float*, const void*, int, void*, int, int64_t, int64_t, const dos_kscal&);
  void (*adam_nta)(float*, float*, float*, const void*, int, void*, int, int64_t, int64_t, const dos_kscal&);
  void (*adam_pf)(float*, float*, float*, const void*, int, void*, int, int64_t, int64_t, const dos_kscal&, int64_t);
};

// H1 through per-thread staging rings (the working copy of host-updated
// subgroups): every team thread updates its contiguous slice of the subgroup
// in chunks of `chunk` elements; a chunk's working copy goes (regular
// stores) into one of the thread's own `nslots` slots, and the thread hands
// it to the shuttle with post() and moves on — no barrier, no CUDA call.  A
// slot is reused only after wait() shows its previous chunk was served.  The
// slots (nslots * chunk * 2 B per thread) stay in the core's L2 / the LLC,
// so the working copy never makes a host-DRAM round trip.
struct dos_ring {
  uint16_t* slots;  // nthreads * nslots * chunk elements, pinned and device-mapped
  int nthreads;     // threads the slots are laid out for (>= the team's)
  int nslots;
  int64_t chunk;
  void* ctx;
  // post: the copy of `count` elements of `slot` to element `offset` of the
  // subgroup's device working copy; returns the shuttle descriptor (>= 0) or
  // a negative DOS_E* code.  wait: block until that descriptor was served.
  int64_t (*post)(void* ctx, const uint16_t* slot, int64_t offset, int64_t count);
  int (*wait)(void* ctx, int64_t id);
};
// `last` (nthreads * nslots entries, -1 = idle) receives each slot's last
// descriptor: the caller waits for them before the subgroup counts as shipped.
int dos_host_adam_ring(float* p, float* m, float* v, const void* g, int gt, int lt, int64_t n, const dos_kscal& s,
                       int nthreads, const dos_ring& ring, int64_t* last);
extern const dos_hk_table dos_hk_avx512;
extern const dos_hk_table dos_hk_avx2;
extern const dos_hk_table dos_hk_generic;

// The shuttle (dos_cuda.cu): a persistent kernel serving copy descriptors
// posted by the host lane into mapped pinned memory (see k_shuttle).
#define DOS_SHUTTLE_Q 1024
struct dos_shuttle_desc {  // 32 B; `id` (= descriptor number + 1) is written last
  uint64_t src, dst;       // device-accessible addresses (host memory: its device alias)
  uint32_t bytes;
  int32_t flag_idx;        // >= 0: flags[flag_idx] = flag_val once the copy has landed
  uint32_t flag_val;
  uint32_t id;
};
struct dos_shuttle_ctl {
  uint32_t stop;           // host: every descriptor of the phase is posted; exit when drained
  uint32_t pad[31];
  uint32_t done[DOS_SHUTTLE_Q];  // kernel: descriptor number + 1 of the last completed one per queue slot
  dos_shuttle_desc q[DOS_SHUTTLE_Q];
};
int dos_shuttle_launch(dos_shuttle_ctl* ctl_dev, uint32_t* flags_dev, uint32_t first, int nctas, cudaStream_t st);
// SMs kept free of K1's persistent grid while a shuttle runs.
void dos_reserve_sms(int n);

// In-phase grad flush through a cache-sized ring (flush_grads): the engine
// pre-enqueues, at CPU_UPDATE submit, the D2H copies of a subgroup's grads
// row by row into `nslots` pinned slots (row = the next `chunk` elements of
// every team thread's slice), each copy gated on the slot's previous row
// having been consumed and followed by a ready flag; the team threads spin on
// the ready flags and read the grads from the slots, which the copy engine
// just wrote (with the host's DMA write-allocate into the LLC they never make
// a DRAM round trip).  Every wait is enqueued at submit time for host work
// emitted earlier, so it stays deadlock-free when streams share a hardware
// queue.
struct dos_gring {
  const uint16_t* slots;   // nslots rows of nthreads * chunk elements
  int nslots;
  int64_t chunk;           // elements per thread per row
  int nthreads;            // the slice layout's thread count
  const uint32_t* ready;   // mapped, per slot: seq + 1 once the row landed
  uint32_t* consumed;      // mapped, per slot: seq + 1 once every thread used the row
  int* counts;             // per slot: threads done with the current row
  uint32_t seq0;           // sequence number of the subgroup's row 0
};
inline int64_t dos_gring_per(int64_t n, int k) { return ((n + k - 1) / k + 63) & ~int64_t(63); }
// rows of a subgroup of n elements (thread 0's slice is the longest)
inline int64_t dos_gring_rows(int64_t n, int k, int64_t chunk) {
  const int64_t per = dos_gring_per(n, k), l0 = per < n ? per : n;
  return (l0 + chunk - 1) / chunk;
}
// threads whose slice has a row c
inline int dos_gring_row_threads(int64_t n, int k, int64_t chunk, int64_t c) {
  const int64_t per = dos_gring_per(n, k);
  int cnt = 0;
  for (int t = 0; t < k; ++t) {
    const int64_t lo = per * t < n ? per * t : n, hi = lo + per < n ? lo + per : n;
    if (lo + c * chunk < hi) ++cnt;
  }
  return cnt;
}
int dos_host_adam_gring(float* p, float* m, float* v, int gt, void* lp, int lt, int64_t n, const dos_kscal& s,
                        const dos_gring& r);
