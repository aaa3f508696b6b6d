// dos_cuda.cu — K1, the sm_100a fused Adam/AdamW kernel of the update phase,
// plus the stand-alone half-precision conversion kernels.
//
// K1 replaces the reference's per-subgroup fast-tier update:
//   ExecutorTarget.apply GPU_UPDATE   (pkg/src/optistate/executor.py:195-205)
//     = upscale(grads16) (core.py:201-205)
//     + adam_step_arrays (kernels.py:107-139 -> _adam_step_jit :88-101)
//   and FLUSH_OUT_MODEL16 = downscale_rne(staged p) (executor.py:219-227),
// fused into ONE pass over HBM: read g (2 B) + p, m, v (12 B), write p, m, v
// (12 B) + the half-precision working copy (2 B) = 28 B/param.
//
// The path is purely HBM-bound (~0.5 flop/B), so there are no tensor cores;
// the design is 128-bit streaming loads/stores (evict-first), 8 elements per
// thread per trip, a grid of resident CTAs sized to the SM count and a
// grid-stride loop.  All arithmetic is IEEE RN without FMA contraction
// (dos_numerics.h), so results are bit-identical to the reference.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>

#include "dos_internal.h"
#include "dos_numerics.h"

namespace {

std::atomic<int64_t> g_launches{0};  // every libdos kernel launch (dos_launch_count)
std::atomic<int> g_reserved_sms{0};  // SMs a running shuttle occupies (K1's persistent grid leaves them out)

constexpr int kThreads = 256;
constexpr int kVec = 8;  // elements per thread per trip

__device__ __forceinline__ void load_g8(const void* g, int gt, int64_t i, float* out) {
  if (gt == DOS_F32) {
    const float4* q = reinterpret_cast<const float4*>(g) + 2 * i;
    const float4 a = __ldcs(q), b = __ldcs(q + 1);
    out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
    out[4] = b.x; out[5] = b.y; out[6] = b.z; out[7] = b.w;
  } else {
    const uint4 w = __ldcs(reinterpret_cast<const uint4*>(g) + i);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint16_t lo = (uint16_t)(ws[k] & 0xffffu), hi = (uint16_t)(ws[k] >> 16);
      if (gt == DOS_BF16) {
        out[2 * k] = dos_bf16_to_f32(lo);
        out[2 * k + 1] = dos_bf16_to_f32(hi);
      } else {
        out[2 * k] = __half2float(__ushort_as_half(lo));  // exact widening
        out[2 * k + 1] = __half2float(__ushort_as_half(hi));
      }
    }
  }
}

__device__ __forceinline__ float load_g1(const void* g, int gt, int64_t i) {
  if (gt == DOS_F32) return reinterpret_cast<const float*>(g)[i];
  const uint16_t b = reinterpret_cast<const uint16_t*>(g)[i];
  return gt == DOS_BF16 ? dos_bf16_to_f32(b) : __half2float(__ushort_as_half(b));
}

__device__ __forceinline__ uint16_t to_lowp(float x, int lt) {
  return lt == DOS_BF16 ? dos_f32_to_bf16(x) : dos_f32_to_f16(x);
}

__device__ __forceinline__ float widen16(uint16_t b, int gt) {
  return gt == DOS_BF16 ? dos_bf16_to_f32(b) : __half2float(__ushort_as_half(b));  // exact
}

// The fused reduce-scatter's rounding (dos_gsrc): the fp32 rank-order sum
// rounded to the grad dtype, then the optional averaging scale, rounded again.
__device__ __forceinline__ float rs_round(float acc, int gt, float scale) {
  uint16_t b = to_lowp(acc, gt);
  if (scale != 1.0f) b = to_lowp(__fmul_rn(widen16(b, gt), scale), gt);
  return widen16(b, gt);
}

// Reduced grad of element e (scalar path).
__device__ __forceinline__ float rs_reduce1(const dos_gsrc& gs, int gt, int64_t e) {
  float acc = widen16(gs.p[0][e], gt);
  for (int r = 1; r < gs.n; ++r) acc = __fadd_rn(acc, widen16(gs.p[r][e], gt));
  return rs_round(acc, gt, gs.scale);
}

// Reduced grads of the 8 elements at base + 8*i (16-byte loads; base + 8*i
// is 16-byte aligned in every source).
__device__ __forceinline__ void rs_reduce8(const dos_gsrc& gs, int gt, int64_t base, int64_t i, float* out) {
#pragma unroll
  for (int r = 0; r < DOS_MAX_PEERS + 1; ++r) {
    if (r >= gs.n) break;
    const uint4 w = __ldcs(reinterpret_cast<const uint4*>(gs.p[r] + base) + i);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float lo = widen16((uint16_t)(ws[k] & 0xffffu), gt), hi = widen16((uint16_t)(ws[k] >> 16), gt);
      out[2 * k] = r ? __fadd_rn(out[2 * k], lo) : lo;
      out[2 * k + 1] = r ? __fadd_rn(out[2 * k + 1], hi) : hi;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) out[k] = rs_round(out[k], gt, gs.scale);
}

// Vector body over [base, base + 8*nvec), plus `nscalar` scalar elements
// (the unaligned head [0, head) and the tail after the vector body).
template <int GT, int LT>
__global__ void __launch_bounds__(kThreads)
    k_adam(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
           const void* g, void* __restrict__ lp, int64_t head, int64_t nvec,
           int64_t n, dos_kscal s, dos_peers pr, dos_gsrc gs) {
  const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * kThreads;

  float* __restrict__ pv = p + head;
  float* __restrict__ mv = m + head;
  float* __restrict__ vv = v + head;
  const char* gv = reinterpret_cast<const char*>(g) + head * (GT == DOS_F32 ? 4 : 2);
  uint16_t* lv = LT == DOS_NONE ? nullptr : reinterpret_cast<uint16_t*>(lp) + head;

  for (int64_t i = tid; i < nvec; i += nthr) {
    float4* P = reinterpret_cast<float4*>(pv) + 2 * i;
    float4* M = reinterpret_cast<float4*>(mv) + 2 * i;
    float4* V = reinterpret_cast<float4*>(vv) + 2 * i;
    const float4 p0 = __ldcs(P), p1 = __ldcs(P + 1);
    const float4 m0 = __ldcs(M), m1 = __ldcs(M + 1);
    const float4 v0 = __ldcs(V), v1 = __ldcs(V + 1);
    float gg[kVec];
    if (GT != DOS_F32 && gs.n > 0) {  // fused reduce-scatter; the reduced grads replace the local ones
      rs_reduce8(gs, GT, head, i, gg);
      uint32_t rw[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) rw[k] = (uint32_t)to_lowp(gg[2 * k], GT) | ((uint32_t)to_lowp(gg[2 * k + 1], GT) << 16);
      __stcs(reinterpret_cast<uint4*>(const_cast<char*>(gv)) + i, make_uint4(rw[0], rw[1], rw[2], rw[3]));
    } else {
      load_g8(gv, GT, i, gg);
    }
    float pe[kVec] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
    float me[kVec] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
    float ve[kVec] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int k = 0; k < kVec; ++k) dos_adam_elem(pe[k], me[k], ve[k], gg[k], s);
    __stcs(P, make_float4(pe[0], pe[1], pe[2], pe[3]));
    __stcs(P + 1, make_float4(pe[4], pe[5], pe[6], pe[7]));
    __stcs(M, make_float4(me[0], me[1], me[2], me[3]));
    __stcs(M + 1, make_float4(me[4], me[5], me[6], me[7]));
    __stcs(V, make_float4(ve[0], ve[1], ve[2], ve[3]));
    __stcs(V + 1, make_float4(ve[4], ve[5], ve[6], ve[7]));
    if (LT != DOS_NONE) {
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        w[k] = (uint32_t)to_lowp(pe[2 * k], LT) | ((uint32_t)to_lowp(pe[2 * k + 1], LT) << 16);
      const uint4 wv = make_uint4(w[0], w[1], w[2], w[3]);
      __stcs(reinterpret_cast<uint4*>(lv) + i, wv);
      for (int r = 0; r < pr.n; ++r) reinterpret_cast<uint4*>(pr.p[r] + head)[i] = wv;  // fused all-gather
    }
  }

  // scalar head + tail
  const int64_t vec_end = head + kVec * nvec;
  const int64_t nscalar = head + (n - vec_end);
  for (int64_t j = tid; j < nscalar; j += nthr) {
    const int64_t e = j < head ? j : vec_end + (j - head);
    float pe = p[e], me = m[e], ve = v[e];
    float ge;
    if (GT != DOS_F32 && gs.n > 0) {
      ge = rs_reduce1(gs, GT, e);
      reinterpret_cast<uint16_t*>(const_cast<void*>(g))[e] = to_lowp(ge, GT);
    } else {
      ge = load_g1(g, GT, e);
    }
    dos_adam_elem(pe, me, ve, ge, s);
    p[e] = pe;
    m[e] = me;
    v[e] = ve;
    if (LT != DOS_NONE) {
      const uint16_t wb = to_lowp(pe, LT);
      reinterpret_cast<uint16_t*>(lp)[e] = wb;
      for (int r = 0; r < pr.n; ++r) pr.p[r][e] = wb;
    }
  }
}

template <int OT>
__global__ void __launch_bounds__(kThreads)
    k_down(const float* __restrict__ x, uint16_t* __restrict__ o, int64_t head, int64_t nvec, int64_t n) {
  const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * kThreads;
  for (int64_t i = tid; i < nvec; i += nthr) {
    const float4* X = reinterpret_cast<const float4*>(x + head) + 2 * i;
    const float4 a = __ldcs(X), b = __ldcs(X + 1);
    const float e[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = (uint32_t)to_lowp(e[2 * k], OT) | ((uint32_t)to_lowp(e[2 * k + 1], OT) << 16);
    __stcs(reinterpret_cast<uint4*>(o + head) + i, make_uint4(w[0], w[1], w[2], w[3]));
  }
  const int64_t vec_end = head + kVec * nvec;
  const int64_t nscalar = head + (n - vec_end);
  for (int64_t j = tid; j < nscalar; j += nthr) {
    const int64_t e = j < head ? j : vec_end + (j - head);
    o[e] = to_lowp(x[e], OT);
  }
}

// Stand-alone reduce-scatter of a range (dos_gsrc rounding): the rank-order
// fp32 sum of every source, rounded to the 16-bit dtype.  Reads 2 B/param
// per rank (all but one over NVLink), writes 2 B/param.
template <int DT>
__global__ void __launch_bounds__(kThreads)
    k_reduce(uint16_t* __restrict__ o, int64_t head, int64_t nvec, int64_t n, dos_gsrc gs) {
  const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * kThreads;
  for (int64_t i = tid; i < nvec; i += nthr) {
    float e[8];
    rs_reduce8(gs, DT, head, i, e);
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = (uint32_t)to_lowp(e[2 * k], DT) | ((uint32_t)to_lowp(e[2 * k + 1], DT) << 16);
    __stcs(reinterpret_cast<uint4*>(o + head) + i, make_uint4(w[0], w[1], w[2], w[3]));
  }
  const int64_t vec_end = head + kVec * nvec;
  const int64_t nscalar = head + (n - vec_end);
  for (int64_t j = tid; j < nscalar; j += nthr) {
    const int64_t e = j < head ? j : vec_end + (j - head);
    o[e] = to_lowp(rs_reduce1(gs, DT, e), DT);
  }
}

template <int IT>
__global__ void __launch_bounds__(kThreads)
    k_up(const uint16_t* __restrict__ x, float* __restrict__ o, int64_t head, int64_t nvec, int64_t n) {
  const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * kThreads;
  for (int64_t i = tid; i < nvec; i += nthr) {
    const uint4 w = __ldcs(reinterpret_cast<const uint4*>(x + head) + i);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    float e[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint16_t lo = (uint16_t)(ws[k] & 0xffffu), hi = (uint16_t)(ws[k] >> 16);
      e[2 * k] = IT == DOS_BF16 ? dos_bf16_to_f32(lo) : dos_f16_to_f32(lo);
      e[2 * k + 1] = IT == DOS_BF16 ? dos_bf16_to_f32(hi) : dos_f16_to_f32(hi);
    }
    float4* O = reinterpret_cast<float4*>(o + head) + 2 * i;
    __stcs(O, make_float4(e[0], e[1], e[2], e[3]));
    __stcs(O + 1, make_float4(e[4], e[5], e[6], e[7]));
  }
  const int64_t vec_end = head + kVec * nvec;
  const int64_t nscalar = head + (n - vec_end);
  for (int64_t j = tid; j < nscalar; j += nthr) {
    const int64_t e = j < head ? j : vec_end + (j - head);
    o[e] = IT == DOS_BF16 ? dos_bf16_to_f32(x[e]) : dos_f16_to_f32(x[e]);
  }
}

// Smallest head h in [0, 8) that puts every stream on a 16-byte boundary
// (fp32 arrays: 4 B/elt, 16-bit arrays: 2 B/elt); -1 if none exists.
int64_t common_head(const void* const* ptrs, const int* elt_bytes, int k, int64_t n) {
  for (int64_t h = 0; h < kVec && h <= n; ++h) {
    bool ok = true;
    for (int j = 0; j < k && ok; ++j)
      ok = ((reinterpret_cast<uintptr_t>(ptrs[j]) + (uintptr_t)(h * elt_bytes[j])) & 15u) == 0;
    if (ok) return h;
  }
  return -1;
}

int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0, c = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && c > 0)
      cached = c;
    else
      cached = 148;
  }
  return cached;
}

// Resident-CTA grid: 8 CTAs of 256 threads per SM covers the register
// budget of K1 (<= 64 regs/thread) at full occupancy; small launches get
// just enough CTAs.
unsigned grid_for(int64_t work) {
  const int64_t cap = (int64_t)sm_count() * 8;
  int64_t want = (work + kThreads - 1) / kThreads;
  if (want < 1) want = 1;
  return (unsigned)(want < cap ? want : cap);
}

template <int GT, int LT>
void launch_adam(float* p, float* m, float* v, const void* g, void* lp, int64_t head, int64_t nvec,
                 int64_t n, const dos_kscal& s, cudaStream_t st, const dos_peers& pr, const dos_gsrc& gs) {
  const int64_t work = nvec > 0 ? nvec : n;
  static int cap_blocks = 0;  // resident CTAs per SM for this instantiation
  if (!cap_blocks) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_adam<GT, LT>, kThreads, 0) != cudaSuccess || b < 1) b = 4;
    cap_blocks = b;
  }
  const int64_t cap = (int64_t)sm_count() * cap_blocks;
  int64_t want = (work + kThreads - 1) / kThreads;
  want = want < 1 ? 1 : (want < cap ? want : cap);
  k_adam<GT, LT><<<(unsigned)want, kThreads, 0, st>>>(p, m, v, g, lp, head, nvec, n, s, pr, gs);
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

// ---------------------------------------------------------------------------
// K1, TMA-pipelined variant (the default for 16-bit grads).
//
// Persistent CTAs (one per SM) stream tiles of TE elements through an
// S-stage shared-memory ring.  Thread 0 is the producer: for each tile it
// arms the stage's mbarrier with the tile's byte count and issues four 1-D
// bulk copies (cp.async.bulk, SASS UBLKCP) for p, m, v, g; S-1 tiles are
// always in flight, decoupling HBM latency from the long IEEE div/sqrt
// chains.  All threads then update the tile in place in shared memory (the
// working copy overwrites the grads' slot), a proxy fence + barrier publish
// the results, and thread 0 bulk-stores p, m, v and the working copy back
// (cp.async.bulk.global.shared::cta, bulk_group).  A stage is refilled only
// after cp.async.bulk.wait_group.read confirms its previous stores have
// drained out of shared memory.
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init1(uint64_t* bar) {  // expected arrivals: one (the producer)
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a stage that never completes (a byte-count bug, a faulted
// copy) traps after ~seconds instead of hanging the GPU — the launch then
// fails with an error the engine reports.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  for (uint32_t spins = 0; !mbar_try_wait(bar, parity); ++spins)
    if (spins > (1u << 26)) __trap();
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
// Streaming variants: the state passes through L2 exactly once, so mark it
// evict-first and leave L2 to the copy engines' traffic of the same phase.
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_load_ef(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_store_ef(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Shared memory of one pipeline stage: p, m, v (fp32), the grads (fp32 or
// 16-bit) and — for fp32 grads only — a separate working-copy slot (16-bit
// grads are overwritten in place by the working copy).
template <int GT, int LT, int NT>
__host__ __device__ constexpr uint32_t tma_stage_bytes() {
  return 4 * NT * (12 + (GT == DOS_F32 ? 4 : 2) + ((GT == DOS_F32 && LT != DOS_NONE) ? 2 : 0));
}

// RS: the grads are the fused reduce-scatter of gs (16-bit grads only).  The
// local rank's tile still arrives by TMA; every other rank's 4 elements of
// this thread come over NVLink as one 8-byte load per rank, issued RD tiles
// ahead (right after a tile's are consumed, the loads of tile k + RD go out)
// so their latency hides behind RD tiles' updates, stores and stage waits.
template <int GT, int LT, int NT, int S, bool RS = false, int RD = 1>
__global__ void __launch_bounds__(NT, 1)
    k_adam_tma(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
               const void* gv, uint16_t* __restrict__ w, int64_t ntiles, int64_t tail,
               dos_kscal s, dos_peers pr, int l2ef, dos_gsrc gs) {
  constexpr int TE = 4 * NT;  // 4 elements per thread per tile
  constexpr uint32_t F32B = TE * 4, H16B = TE * 2, GB = GT == DOS_F32 ? F32B : H16B;
  constexpr uint32_t STAGE = tma_stage_bytes<GT, LT, NT>();
  constexpr uint32_t WOFF = GT == DOS_F32 ? 3 * F32B + GB : 3 * F32B;  // working-copy slot
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[S];
  const int tid = threadIdx.x;
  const int64_t first = blockIdx.x, step = gridDim.x;
  const int64_t mine = ntiles > first ? (ntiles - first + step - 1) / step : 0;
  const uint64_t pol = l2ef ? l2_evict_first() : 0;
  const char* g = static_cast<const char*>(gv);
  constexpr int GE = GT == DOS_F32 ? 4 : 2;  // bytes per grad element

  auto stage_ptr = [&](int st, int piece) -> unsigned char* {
    return smem + st * STAGE + (piece == 4 ? WOFF : piece * F32B);
  };
  auto load = [&](void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    if (l2ef) bulk_load_ef(dst, src, bytes, bar, pol);
    else bulk_load(dst, src, bytes, bar);
  };
  auto store = [&](void* dst, const void* src, uint32_t bytes) {
    if (l2ef) bulk_store_ef(dst, src, bytes, pol);
    else bulk_store(dst, src, bytes);
  };
  auto issue = [&](int64_t k) {  // tile k of this CTA into stage k % S
    const int st = (int)(k % S);
    const int64_t e0 = (first + k * step) * TE;
    mbar_expect_tx(&full[st], 3 * F32B + GB);  // the bytes the four loads deliver (not the W slot)
    load(stage_ptr(st, 0), p + e0, F32B, &full[st]);
    load(stage_ptr(st, 1), m + e0, F32B, &full[st]);
    load(stage_ptr(st, 2), v + e0, F32B, &full[st]);
    load(stage_ptr(st, 3), g + e0 * GE, GB, &full[st]);
  };

  if (tid == 0) {
    for (int i = 0; i < S; ++i) mbar_init1(&full[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");  // inits visible to the async proxy
    fence_async_smem();
  }
  __syncthreads();
  if (tid == 0)
    for (int64_t k = 0; k < S - 1 && k < mine; ++k) issue(k);

  // RS: the other ranks' grads of the next RD tiles, a register queue
  // (nx[0] = the tile being updated; static indices only, so no local memory)
  uint2 nx[RS ? RD : 1][RS ? DOS_MAX_PEERS + 1 : 1];
  auto rs_fetch = [&](int64_t k, int slot) {
    const int64_t e0 = (first + k * step) * TE;
#pragma unroll
    for (int q = 0; q < (RS ? RD : 0); ++q)
      if (q == slot) {
#pragma unroll
        for (int r = 0; r < (RS ? DOS_MAX_PEERS + 1 : 0); ++r)
          if (r < gs.n && r != gs.self) nx[q][r] = __ldcs(reinterpret_cast<const uint2*>(gs.p[r] + e0) + tid);
      }
  };
  if (RS) {
#pragma unroll
    for (int q = 0; q < RD; ++q)
      if (q < mine) rs_fetch(q, q);
  }

  for (int64_t k = 0; k < mine; ++k) {
    const int st = (int)(k % S);
    mbar_wait(&full[st], (uint32_t)((k / S) & 1));
    float4* P = reinterpret_cast<float4*>(stage_ptr(st, 0)) + tid;
    float4* M = reinterpret_cast<float4*>(stage_ptr(st, 1)) + tid;
    float4* V = reinterpret_cast<float4*>(stage_ptr(st, 2)) + tid;
    float4 pp = *P, mm = *M, vv = *V;
    float pe[4] = {pp.x, pp.y, pp.z, pp.w}, me[4] = {mm.x, mm.y, mm.z, mm.w}, ve[4] = {vv.x, vv.y, vv.z, vv.w};
    float ge[4];
    if (GT == DOS_F32) {
      const float4 gg = reinterpret_cast<const float4*>(stage_ptr(st, 3))[tid];
      ge[0] = gg.x; ge[1] = gg.y; ge[2] = gg.z; ge[3] = gg.w;
    } else {
      const uint2 gg = reinterpret_cast<const uint2*>(stage_ptr(st, 3))[tid];
      const uint16_t gb[4] = {(uint16_t)(gg.x & 0xffffu), (uint16_t)(gg.x >> 16), (uint16_t)(gg.y & 0xffffu),
                              (uint16_t)(gg.y >> 16)};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        ge[j] = GT == DOS_BF16 ? dos_bf16_to_f32(gb[j]) : __half2float(__ushort_as_half(gb[j]));
      if (RS) {  // rank-order fp32 sum with the local tile at position gs.self
        float acc[4];
#pragma unroll
        for (int r = 0; r < DOS_MAX_PEERS + 1; ++r) {
          if (r >= gs.n) break;
          float x[4];
          if (r == gs.self) {
            x[0] = ge[0]; x[1] = ge[1]; x[2] = ge[2]; x[3] = ge[3];
          } else {
            x[0] = widen16((uint16_t)(nx[0][r].x & 0xffffu), GT);
            x[1] = widen16((uint16_t)(nx[0][r].x >> 16), GT);
            x[2] = widen16((uint16_t)(nx[0][r].y & 0xffffu), GT);
            x[3] = widen16((uint16_t)(nx[0][r].y >> 16), GT);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[j] = r ? __fadd_rn(acc[j], x[j]) : x[j];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) ge[j] = rs_round(acc[j], GT, gs.scale);
        // shift the queue and put tile k + RD's loads in flight
#pragma unroll
        for (int q = 0; q + 1 < RD; ++q)
#pragma unroll
          for (int r = 0; r < DOS_MAX_PEERS + 1; ++r) nx[q][r] = nx[q + 1][r];
        if (k + RD < mine) rs_fetch(k + RD, RD - 1);
        // the reduced grads replace the local ones (as an NCCL reduce-scatter would leave them)
        const int64_t e0 = (first + k * step) * TE;
        __stcs(reinterpret_cast<uint2*>(const_cast<char*>(g) + e0 * GE) + tid,
               make_uint2((uint32_t)to_lowp(ge[0], GT) | ((uint32_t)to_lowp(ge[1], GT) << 16),
                          (uint32_t)to_lowp(ge[2], GT) | ((uint32_t)to_lowp(ge[3], GT) << 16)));
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) dos_adam_elem(pe[j], me[j], ve[j], ge[j], s);
    *P = make_float4(pe[0], pe[1], pe[2], pe[3]);
    *M = make_float4(me[0], me[1], me[2], me[3]);
    *V = make_float4(ve[0], ve[1], ve[2], ve[3]);
    if (LT != DOS_NONE) {
      const uint2 wv = make_uint2((uint32_t)to_lowp(pe[0], LT) | ((uint32_t)to_lowp(pe[1], LT) << 16),
                                  (uint32_t)to_lowp(pe[2], LT) | ((uint32_t)to_lowp(pe[3], LT) << 16));
      reinterpret_cast<uint2*>(stage_ptr(st, 4))[tid] = wv;
      // fused all-gather: the same 8 bytes straight into every peer's copy
      // (NVLink stores through IPC-mapped addresses), coalesced per warp
      const int64_t e0 = (first + k * step) * TE;
      for (int r = 0; r < pr.n; ++r) reinterpret_cast<uint2*>(pr.p[r] + e0)[tid] = wv;
    }
    fence_async_smem();  // generic-proxy smem writes -> visible to the bulk-copy (async) proxy
    __syncthreads();
    if (tid == 0) {
      const int64_t e0 = (first + k * step) * TE;
      store(p + e0, stage_ptr(st, 0), F32B);
      store(m + e0, stage_ptr(st, 1), F32B);
      store(v + e0, stage_ptr(st, 2), F32B);
      if (LT != DOS_NONE) store(w + e0, stage_ptr(st, 4), H16B);
      bulk_commit();
      if (k + S - 1 < mine) {
        bulk_wait_read<1>();  // the refilled stage's stores (tile k-1) have left shared memory
        issue(k + S - 1);
      }
    }
  }
  // the ragged tail (< one tile) after the last tile: the last CTA, straight
  // from global memory, so a subgroup is one launch
  if (blockIdx.x == gridDim.x - 1) {
    const int64_t base = ntiles * TE;
    for (int64_t j = tid; j < tail; j += NT) {
      const int64_t e = base + j;
      float pe = p[e], me = m[e], ve = v[e];
      const float gj = RS ? rs_reduce1(gs, GT, e) : load_g1(gv, GT, e);
      if (RS) reinterpret_cast<uint16_t*>(const_cast<void*>(gv))[e] = to_lowp(gj, GT);
      dos_adam_elem(pe, me, ve, gj, s);
      p[e] = pe;
      m[e] = me;
      v[e] = ve;
      if (LT != DOS_NONE) {
        const uint16_t wb = to_lowp(pe, LT);
        w[e] = wb;
        for (int r = 0; r < pr.n; ++r) pr.p[r][e] = wb;
      }
    }
  }
  if (tid == 0) bulk_wait_all();
}

template <int GT, int LT, int NT, int S, bool RS = false, int RD = 1>
int launch_tma_cfg(float* p, float* m, float* v, const void* g, uint16_t* w, int64_t ntiles, int64_t tail,
                   const dos_kscal& s, int ctas_per_sm, cudaStream_t st, const dos_peers& pr,
                   const dos_gsrc& gs = dos_gsrc{0, 0, 1.0f, {}}) {
  constexpr int smem = S * tma_stage_bytes<GT, LT, NT>();
  static bool configured = false;
  if (!configured) {
    const cudaError_t e =
        cudaFuncSetAttribute(k_adam_tma<GT, LT, NT, S, RS, RD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return dos_set_error(DOS_ECUDA, "K1 smem attribute: %s", cudaGetErrorString(e));
    configured = true;
  }
  const int64_t cap = (int64_t)std::max(1, sm_count() - g_reserved_sms.load(std::memory_order_relaxed)) * ctas_per_sm;
  const int64_t grid = ntiles < cap ? ntiles : cap;
  // DOS_K1_L2=evict_first turns on L2 evict-first hints for the bulk copies;
  // measured on the B200 they do not help (alone or under duplex DMA), so off.
  static const int l2ef = [] {
    const char* e = getenv("DOS_K1_L2");
    return (e && strcmp(e, "evict_first") == 0) ? 1 : 0;
  }();
  k_adam_tma<GT, LT, NT, S, RS, RD><<<(unsigned)grid, NT, smem, st>>>(p, m, v, g, w, ntiles, tail, s, pr, l2ef, gs);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return DOS_OK;
}

// Pipeline shapes (threads, stages, CTAs/SM); tile = 4 x threads elements,
// 14 B/element of shared memory per stage.  DOS_K1_CFG=<index> selects one
// for A/B sweeps; DOS_K1=ldg forces the register path.
struct TmaCfg {
  int nt, stages, cpb;
};
// Index 0 is the default: 1024 threads, 3 x 56 KB stages, one CTA per SM
// (swept on the B200: profiles/k1_pipeline_sweep.json).
constexpr TmaCfg kTmaCfgs[] = {{1024, 3, 1}, {512, 6, 1}, {256, 12, 1}, {256, 6, 2}, {512, 3, 2},
                               {128, 12, 2}, {1024, 4, 1}, {1024, 2, 2}, {512, 4, 2}};

const TmaCfg& tma_cfg() {
  static int idx = -1;
  if (idx < 0) {
    const char* e = getenv("DOS_K1_CFG");
    idx = e ? atoi(e) : 0;
    if (idx < 0 || idx >= (int)(sizeof(kTmaCfgs) / sizeof(kTmaCfgs[0]))) idx = 0;
  }
  return kTmaCfgs[idx];
}

bool tma_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("DOS_K1");
    on = (e && strcmp(e, "ldg") == 0) ? 0 : 1;
  }
  return on == 1;
}

// Does the selected pipeline shape fit in a CTA's shared memory for these dtypes?
bool tma_fits(int gt, int lt) {
  const TmaCfg& c = tma_cfg();
  const int per_elem = 12 + (gt == DOS_F32 ? 4 : 2) + ((gt == DOS_F32 && lt != DOS_NONE) ? 2 : 0);
  return (int64_t)c.stages * 4 * c.nt * per_elem <= 227 * 1024;
}

template <int GT, int LT>
int launch_adam_tma(float* p, float* m, float* v, const void* g, uint16_t* w, int64_t ntiles, int64_t tail,
                    const dos_kscal& s, cudaStream_t st, const dos_peers& pr) {
  const TmaCfg& c = tma_cfg();
#define DOS_CFG(NT_, S_) \
  if (c.nt == NT_ && c.stages == S_)  \
    return launch_tma_cfg<GT, LT, NT_, S_>(p, m, v, g, w, ntiles, tail, s, c.cpb, st, pr);
  DOS_CFG(1024, 3)
  DOS_CFG(512, 6)
  DOS_CFG(256, 12)
  DOS_CFG(256, 6)
  DOS_CFG(512, 3)
  DOS_CFG(128, 12)
  DOS_CFG(1024, 4)
  DOS_CFG(1024, 2)
  DOS_CFG(512, 4)
#undef DOS_CFG
  return dos_set_error(DOS_EINVAL, "no K1 pipeline shape %d/%d", c.nt, c.stages);
}

// Fused reduce-scatter pipeline: shape (threads, stages, CTAs/SM) and how
// many tiles ahead the peers' grads are loaded.  DOS_K1_RS=<shape>,<depth>:
// shape 0 = 1024 x 3 x 1 (default), 1 = 512 x 6 x 1 (deeper TMA ring, more
// registers per thread for the peer queue); depth 1 (default) or 2.
// Swept with tools/k1_rs.py (profiles/r02_k1_rs_depth_shape.json).
struct RsCfg {
  int nt, stages, cpb, depth;
};
const RsCfg& rs_cfg() {
  static RsCfg c = [] {
    RsCfg r{1024, 3, 1, 1};
    const char* e = getenv("DOS_K1_RS");
    if (e) {
      int shape = 0, depth = 1;
      if (sscanf(e, "%d,%d", &shape, &depth) >= 1) {
        if (shape == 1) r = RsCfg{512, 6, 1, 1};
        r.depth = depth == 2 ? 2 : 1;
      }
    }
    return r;
  }();
  return c;
}

template <int G, int L>
int launch_rs_shape(float* p, float* m, float* v, const void* g, uint16_t* w, int64_t ntiles, int64_t tail,
                    const dos_kscal& s, cudaStream_t st, const dos_peers& pr, const dos_gsrc& gs) {
  const RsCfg& c = rs_cfg();
  if (c.nt == 1024)
    return c.depth == 2 ? launch_tma_cfg<G, L, 1024, 3, true, 2>(p, m, v, g, w, ntiles, tail, s, c.cpb, st, pr, gs)
                        : launch_tma_cfg<G, L, 1024, 3, true, 1>(p, m, v, g, w, ntiles, tail, s, c.cpb, st, pr, gs);
  return c.depth == 2 ? launch_tma_cfg<G, L, 512, 6, true, 2>(p, m, v, g, w, ntiles, tail, s, c.cpb, st, pr, gs)
                      : launch_tma_cfg<G, L, 512, 6, true, 1>(p, m, v, g, w, ntiles, tail, s, c.cpb, st, pr, gs);
}

int launch_adam_tma_rs(int gt, int lt, float* p, float* m, float* v, const void* g, uint16_t* w, int64_t ntiles,
                       int64_t tail, const dos_kscal& s, cudaStream_t st, const dos_peers& pr, const dos_gsrc& gs) {
  if (gt == DOS_BF16 && lt == DOS_BF16) return launch_rs_shape<DOS_BF16, DOS_BF16>(p, m, v, g, w, ntiles, tail, s, st, pr, gs);
  if (gt == DOS_F16 && lt == DOS_F16) return launch_rs_shape<DOS_F16, DOS_F16>(p, m, v, g, w, ntiles, tail, s, st, pr, gs);
  if (gt == DOS_BF16 && lt == DOS_NONE) return launch_rs_shape<DOS_BF16, DOS_NONE>(p, m, v, g, w, ntiles, tail, s, st, pr, gs);
  if (gt == DOS_F16 && lt == DOS_NONE) return launch_rs_shape<DOS_F16, DOS_NONE>(p, m, v, g, w, ntiles, tail, s, st, pr, gs);
  return dos_set_error(DOS_ETYPE, "fused reduce-scatter: working copy must match the grad dtype (g=%d lowp=%d)", gt, lt);
}

}  // namespace

dos_kscal dos_make_kscal(const dos_adam_scalars* s) {
  dos_kscal k;
  k.lr = s->lr;
  k.b1 = s->beta1;
  k.b2 = s->beta2;
  k.eps = s->eps;
  k.bc1 = s->bc1;
  k.bc2 = s->bc2;
  volatile float one = 1.0f;  // fp32 difference, as np.float32(1) - np.float32(beta)
  k.omb1 = one - s->beta1;
  k.omb2 = one - s->beta2;
  volatile float lrwd = s->lr * s->weight_decay;
  k.decay = one - lrwd;
  k.adamw = s->adamw != 0;
  return k;
}

dos_peers dos_peers_offset(const dos_peers& pr, int64_t elems) {
  dos_peers o = pr;
  for (int r = 0; r < pr.n; ++r) o.p[r] = pr.p[r] + elems;
  return o;
}

dos_gsrc dos_gsrc_offset(const dos_gsrc& gs, int64_t elems) {
  dos_gsrc o = gs;
  for (int r = 0; r < gs.n; ++r) o.p[r] = gs.p[r] + elems;
  return o;
}

int dos_adam_launch(float* p, float* m, float* v, const void* g, int gt, void* lp, int lt, int64_t n,
                    const dos_kscal& s, cudaStream_t st, const dos_peers& pr, const dos_gsrc& gs) {
  if (n == 0) return DOS_OK;
  if (pr.n > 0 && lt == DOS_NONE) return dos_set_error(DOS_EINVAL, "peer broadcast needs a working-copy dtype");
  if (gs.n > 0 && gt == DOS_F32) return dos_set_error(DOS_ETYPE, "the fused reduce-scatter takes 16-bit grads");
  const void* ptrs[5 + 2 * DOS_MAX_PEERS + 1] = {p, m, v, g, lp};
  int eb[5 + 2 * DOS_MAX_PEERS + 1] = {4, 4, 4, gt == DOS_F32 ? 4 : 2, 2};
  int k = 5;
  for (int r = 0; r < pr.n; ++r, ++k) {  // peers share the 16-byte phase of the local stores
    ptrs[k] = pr.p[r];
    eb[k] = 2;
  }
  for (int r = 0; r < gs.n; ++r, ++k) {  // and so do the reduce-scatter's sources
    ptrs[k] = gs.p[r];
    eb[k] = 2;
  }
  if (lt == DOS_NONE) {  // no working copy: drop lp from the alignment set
    for (int j = 4; j + 1 < k; ++j) {
      ptrs[j] = ptrs[j + 1];
      eb[j] = eb[j + 1];
    }
    --k;
  }
  int64_t head = common_head(ptrs, eb, k, n);
  // TMA path: a 16-byte-alignable range of at least one tile whose pipeline
  // shape fits in shared memory (all grad dtypes).  The fused reduce-scatter
  // always uses the default shape (1024 threads x 3 stages, one CTA per SM).
  const int64_t tile = gs.n > 0 ? 4 * rs_cfg().nt : 4 * tma_cfg().nt;
  if ((gt == DOS_F32 || gt == DOS_F16 || gt == DOS_BF16) && (lt == DOS_NONE || lt == DOS_F16 || lt == DOS_BF16) &&
      head >= 0 && tma_enabled() && (gs.n > 0 || tma_fits(gt, lt)) && (n - head) / tile >= 1) {
    const int64_t ntiles = (n - head) / tile;
    const int64_t tail = n - head - ntiles * tile;  // < one tile; handled inside the same launch
    const char* gc = static_cast<const char*>(g);
    char* lc = static_cast<char*>(lp);
    int rc = DOS_OK;
    if (head > 0) rc = dos_adam_launch(p, m, v, g, gt, lp, lt, head, s, st, pr, gs);  // < 8 elements: register path
    if (rc != DOS_OK) return rc;
    const void* gb = gc + (gt == DOS_F32 ? 4 : 2) * head;
    uint16_t* wb = lt == DOS_NONE ? nullptr : reinterpret_cast<uint16_t*>(lc + 2 * head);
    const dos_peers pb = dos_peers_offset(pr, head);
    if (gs.n > 0) {
      rc = launch_adam_tma_rs(gt, lt, p + head, m + head, v + head, gb, wb, ntiles, tail, s, st, pb,
                              dos_gsrc_offset(gs, head));
      if (rc != DOS_OK) return rc;
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return dos_set_error(DOS_ECUDA, "K1 (TMA, RS) launch failed: %s", cudaGetErrorString(e));
      return DOS_OK;
    }
#define DOS_TMA(G, L) \
  if (gt == G && lt == L) rc = launch_adam_tma<G, L>(p + head, m + head, v + head, gb, wb, ntiles, tail, s, st, pb);
    DOS_TMA(DOS_F16, DOS_NONE) else DOS_TMA(DOS_F16, DOS_F16) else DOS_TMA(DOS_F16, DOS_BF16)
    else DOS_TMA(DOS_BF16, DOS_NONE) else DOS_TMA(DOS_BF16, DOS_F16) else DOS_TMA(DOS_BF16, DOS_BF16)
    else DOS_TMA(DOS_F32, DOS_NONE) else DOS_TMA(DOS_F32, DOS_F16) else DOS_TMA(DOS_F32, DOS_BF16)
#undef DOS_TMA
    if (rc != DOS_OK) return rc;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return dos_set_error(DOS_ECUDA, "K1 (TMA) launch failed: %s", cudaGetErrorString(e));
    return rc;
  }
  int64_t nvec = 0;
  if (head < 0) {
    head = n;  // no common alignment: everything takes the scalar path
  } else {
    nvec = (n - head) / kVec;
  }
#define DOS_CASE(G, L) \
  if (gt == G && lt == L) { launch_adam<G, L>(p, m, v, g, lp, head, nvec, n, s, st, pr, gs); }
  DOS_CASE(DOS_F32, DOS_NONE) else DOS_CASE(DOS_F32, DOS_F16) else DOS_CASE(DOS_F32, DOS_BF16)
  else DOS_CASE(DOS_F16, DOS_NONE) else DOS_CASE(DOS_F16, DOS_F16) else DOS_CASE(DOS_F16, DOS_BF16)
  else DOS_CASE(DOS_BF16, DOS_NONE) else DOS_CASE(DOS_BF16, DOS_F16) else DOS_CASE(DOS_BF16, DOS_BF16)
  else return dos_set_error(DOS_ETYPE, "unsupported dtype pair g=%d lowp=%d", gt, lt);
#undef DOS_CASE
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dos_set_error(DOS_ECUDA, "K1 launch failed: %s", cudaGetErrorString(e));
  return DOS_OK;
}

extern "C" int dos_adam_step_cuda(float* p, float* m, float* v, const void* g, int g_dtype, void* p_lowp,
                                  int lowp_dtype, int64_t n, const dos_adam_scalars* s, void* stream) {
  if (!s) return dos_set_error(DOS_EINVAL, "scalars must not be NULL");
  if (n < 0) return dos_set_error(DOS_EINVAL, "n must be >= 0");
  if (g_dtype != DOS_F32 && g_dtype != DOS_F16 && g_dtype != DOS_BF16)
    return dos_set_error(DOS_ETYPE, "grad dtype %d unsupported", g_dtype);
  if (lowp_dtype != DOS_NONE && lowp_dtype != DOS_F16 && lowp_dtype != DOS_BF16)
    return dos_set_error(DOS_ETYPE, "working-copy dtype %d unsupported", lowp_dtype);
  if (n > 0 && (!p || !m || !v || !g || (lowp_dtype != DOS_NONE && !p_lowp)))
    return dos_set_error(DOS_EINVAL, "NULL buffer");
  return dos_adam_launch(p, m, v, g, g_dtype, p_lowp, lowp_dtype, n, dos_make_kscal(s),
                         reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int dos_adam_step_cuda_bcast(float* p, float* m, float* v, const void* g, int g_dtype, void* p_lowp,
                                        int lowp_dtype, void* const* peer_lowp, int npeers, int64_t n,
                                        const dos_adam_scalars* s, void* stream) {
  if (npeers < 0 || npeers > DOS_MAX_PEERS) return dos_set_error(DOS_EINVAL, "npeers must be in [0, %d]", DOS_MAX_PEERS);
  if (npeers > 0 && (lowp_dtype == DOS_NONE || !peer_lowp)) return dos_set_error(DOS_EINVAL, "peers need a working copy");
  if (!s) return dos_set_error(DOS_EINVAL, "scalars must not be NULL");
  if (n < 0) return dos_set_error(DOS_EINVAL, "n must be >= 0");
  if (g_dtype != DOS_F32 && g_dtype != DOS_F16 && g_dtype != DOS_BF16)
    return dos_set_error(DOS_ETYPE, "grad dtype %d unsupported", g_dtype);
  if (lowp_dtype != DOS_NONE && lowp_dtype != DOS_F16 && lowp_dtype != DOS_BF16)
    return dos_set_error(DOS_ETYPE, "working-copy dtype %d unsupported", lowp_dtype);
  if (n > 0 && (!p || !m || !v || !g || (lowp_dtype != DOS_NONE && !p_lowp)))
    return dos_set_error(DOS_EINVAL, "NULL buffer");
  dos_peers pr{npeers, {}};
  for (int r = 0; r < npeers; ++r) {
    if (!peer_lowp[r]) return dos_set_error(DOS_EINVAL, "NULL peer pointer %d", r);
    pr.p[r] = static_cast<uint16_t*>(peer_lowp[r]);
  }
  return dos_adam_launch(p, m, v, g, g_dtype, p_lowp, lowp_dtype, n, dos_make_kscal(s),
                         reinterpret_cast<cudaStream_t>(stream), pr);
}

extern "C" int dos_downscale_cuda(const float* x, void* out, int out_dtype, int64_t n, void* stream) {
  if (n < 0) return dos_set_error(DOS_EINVAL, "n must be >= 0");
  if (out_dtype != DOS_F16 && out_dtype != DOS_BF16)
    return dos_set_error(DOS_ETYPE, "downscale target dtype %d unsupported", out_dtype);
  if (n == 0) return DOS_OK;
  const void* ptrs[2] = {x, out};
  const int eb[2] = {4, 2};
  int64_t head = common_head(ptrs, eb, 2, n), nvec = 0;
  if (head < 0) head = n; else nvec = (n - head) / kVec;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const unsigned grid = grid_for(nvec > 0 ? nvec : n);
  if (out_dtype == DOS_F16)
    k_down<DOS_F16><<<grid, kThreads, 0, st>>>(x, reinterpret_cast<uint16_t*>(out), head, nvec, n);
  else
    k_down<DOS_BF16><<<grid, kThreads, 0, st>>>(x, reinterpret_cast<uint16_t*>(out), head, nvec, n);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dos_set_error(DOS_ECUDA, "downscale launch failed: %s", cudaGetErrorString(e));
  return DOS_OK;
}

extern "C" int dos_upscale_cuda(const void* x, int in_dtype, float* out, int64_t n, void* stream) {
  if (n < 0) return dos_set_error(DOS_EINVAL, "n must be >= 0");
  if (in_dtype != DOS_F16 && in_dtype != DOS_BF16)
    return dos_set_error(DOS_ETYPE, "upscale source dtype %d unsupported", in_dtype);
  if (n == 0) return DOS_OK;
  const void* ptrs[2] = {x, out};
  const int eb[2] = {2, 4};
  int64_t head = common_head(ptrs, eb, 2, n), nvec = 0;
  if (head < 0) head = n; else nvec = (n - head) / kVec;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const unsigned grid = grid_for(nvec > 0 ? nvec : n);
  if (in_dtype == DOS_F16)
    k_up<DOS_F16><<<grid, kThreads, 0, st>>>(reinterpret_cast<const uint16_t*>(x), out, head, nvec, n);
  else
    k_up<DOS_BF16><<<grid, kThreads, 0, st>>>(reinterpret_cast<const uint16_t*>(x), out, head, nvec, n);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dos_set_error(DOS_ECUDA, "upscale launch failed: %s", cudaGetErrorString(e));
  return DOS_OK;
}

extern "C" int64_t dos_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int dos_reduce_launch(void* out, int dt, int64_t n, const dos_gsrc& gs, cudaStream_t st) {
  if (n == 0) return DOS_OK;
  if (dt != DOS_F16 && dt != DOS_BF16) return dos_set_error(DOS_ETYPE, "reduce-scatter dtype %d unsupported", dt);
  if (gs.n < 1 || gs.n > DOS_MAX_PEERS + 1) return dos_set_error(DOS_EINVAL, "reduce-scatter needs 1..%d sources", DOS_MAX_PEERS + 1);
  const void* ptrs[DOS_MAX_PEERS + 2] = {out};
  int eb[DOS_MAX_PEERS + 2] = {2};
  for (int r = 0; r < gs.n; ++r) {
    ptrs[1 + r] = gs.p[r];
    eb[1 + r] = 2;
  }
  int64_t head = common_head(ptrs, eb, 1 + gs.n, n), nvec = 0;
  if (head < 0) head = n; else nvec = (n - head) / kVec;
  const unsigned grid = grid_for(nvec > 0 ? nvec : n);
  uint16_t* o = static_cast<uint16_t*>(out);
  if (dt == DOS_F16) k_reduce<DOS_F16><<<grid, kThreads, 0, st>>>(o, head, nvec, n, gs);
  else k_reduce<DOS_BF16><<<grid, kThreads, 0, st>>>(o, head, nvec, n, gs);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dos_set_error(DOS_ECUDA, "reduce-scatter launch failed: %s", cudaGetErrorString(e));
  return DOS_OK;
}

namespace {
int make_gsrc(const void* const* src, int nsrc, int self, float scale, dos_gsrc* out) {
  if (nsrc < 1 || nsrc > DOS_MAX_PEERS + 1 || !src)
    return dos_set_error(DOS_EINVAL, "nsrc must be in [1, %d] with source pointers", DOS_MAX_PEERS + 1);
  if (self < 0 || self >= nsrc) return dos_set_error(DOS_EINVAL, "self rank %d outside [0, %d)", self, nsrc);
  if (!(scale > 0.0f) || scale != scale) return dos_set_error(DOS_EINVAL, "grad scale must be positive");
  out->n = nsrc;
  out->self = self;
  out->scale = scale;
  for (int r = 0; r < nsrc; ++r) {
    if (!src[r]) return dos_set_error(DOS_EINVAL, "NULL grad source %d", r);
    out->p[r] = static_cast<const uint16_t*>(src[r]);
  }
  return DOS_OK;
}
}  // namespace

extern "C" int dos_reduce_scatter_cuda(void* out, const void* const* src, int nsrc, int dtype, float scale,
                                       int64_t n, void* stream) {
  if (n < 0) return dos_set_error(DOS_EINVAL, "n must be >= 0");
  if (dtype != DOS_F16 && dtype != DOS_BF16) return dos_set_error(DOS_ETYPE, "reduce-scatter dtype %d unsupported", dtype);
  if (n > 0 && !out) return dos_set_error(DOS_EINVAL, "NULL output");
  dos_gsrc gs;
  const int rc = make_gsrc(src, nsrc, 0, scale, &gs);
  if (rc != DOS_OK) return rc;
  return dos_reduce_launch(out, dtype, n, gs, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int dos_adam_step_cuda_rs(float* p, float* m, float* v, const void* const* g_src, int nsrc, int self,
                                     int g_dtype, float grad_scale, void* p_lowp, int lowp_dtype,
                                     void* const* peer_lowp, int npeers, int64_t n, const dos_adam_scalars* s,
                                     void* stream) {
  if (!s) return dos_set_error(DOS_EINVAL, "scalars must not be NULL");
  if (n < 0) return dos_set_error(DOS_EINVAL, "n must be >= 0");
  if (g_dtype != DOS_F16 && g_dtype != DOS_BF16)
    return dos_set_error(DOS_ETYPE, "the fused reduce-scatter takes 16-bit grads (dtype %d)", g_dtype);
  if (lowp_dtype != DOS_NONE && lowp_dtype != g_dtype)
    return dos_set_error(DOS_ETYPE, "working copy dtype %d must match the grads (%d)", lowp_dtype, g_dtype);
  if (npeers < 0 || npeers > DOS_MAX_PEERS) return dos_set_error(DOS_EINVAL, "npeers must be in [0, %d]", DOS_MAX_PEERS);
  if (npeers > 0 && (lowp_dtype == DOS_NONE || !peer_lowp)) return dos_set_error(DOS_EINVAL, "peers need a working copy");
  if (n > 0 && (!p || !m || !v || (lowp_dtype != DOS_NONE && !p_lowp))) return dos_set_error(DOS_EINVAL, "NULL buffer");
  dos_gsrc gs;
  int rc = make_gsrc(g_src, nsrc, self, grad_scale, &gs);
  if (rc != DOS_OK) return rc;
  dos_peers pr{npeers, {}};
  for (int r = 0; r < npeers; ++r) {
    if (!peer_lowp[r]) return dos_set_error(DOS_EINVAL, "NULL peer pointer %d", r);
    pr.p[r] = static_cast<uint16_t*>(peer_lowp[r]);
  }
  return dos_adam_launch(p, m, v, gs.p[self], g_dtype, p_lowp, lowp_dtype, n, dos_make_kscal(s),
                         reinterpret_cast<cudaStream_t>(stream), pr, gs);
}

// ---------------------------------------------------------------- coherence
// The reference's post-phase guarantee (executor.py:271-282): every
// subgroup's half-precision params equal downscale(params32), bit for bit.
// One launch checks a batch of ranges; each range is read in `nwin` windows
// of `window` elements — contiguous (the whole range) when nwin*window >= n,
// else spread evenly from the first element to the last (a sample).  p32 and
// the working copy may live in HBM or in mapped pinned host memory (device
// aliases resolved by the caller).  Mismatches are counted in out[0] and the
// smallest (range << 40 | element) key is kept in out[1].
namespace {
constexpr int kCohMax = 160;  // ranges per launch (7.7 KB of kernel parameters)
struct coh_batch {
  int n;
  int lt;
  int base;  // index of range 0 of this batch in the caller's list
  const float* p[kCohMax];
  const uint16_t* w[kCohMax];
  int64_t len[kCohMax], win[kCohMax], nwin[kCohMax], first[kCohMax + 1];
};

__global__ void __launch_bounds__(kThreads) k_coherence(const __grid_constant__ coh_batch b,
                                                         unsigned long long* out) {
  const int64_t total = b.first[b.n];
  for (int64_t pair = blockIdx.x; pair < total; pair += gridDim.x) {
    int lo = 0, hi = b.n - 1;  // range r with first[r] <= pair < first[r+1]
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (b.first[mid] <= pair) lo = mid; else hi = mid - 1;
    }
    const int r = lo;
    const int64_t k = pair - b.first[r], n = b.len[r], win = b.win[r], nw = b.nwin[r];
    const int64_t start = nw * win >= n ? k * win : (nw > 1 ? k * (n - win) / (nw - 1) : 0);
    const int64_t stop = start + win < n ? start + win : n;
    unsigned long long bad = 0, key = ~0ull;
    const float* P = b.p[r];
    const uint16_t* W = b.w[r];
    auto check = [&](float x, uint16_t y, int64_t i) {
      if (to_lowp(x, b.lt) != y) {
        ++bad;
        const unsigned long long kk = ((unsigned long long)(b.base + r) << 40) | (unsigned long long)i;
        key = kk < key ? kk : key;
      }
    };
    int64_t i0 = start;
    // 4 elements per load (16 B of p32, 8 B of working copy) where both align
    if ((((uintptr_t)(P + start)) & 15u) == 0 && (((uintptr_t)(W + start)) & 7u) == 0) {
      const int64_t nv = (stop - start) / 4;
      const float4* P4 = reinterpret_cast<const float4*>(P + start);
      const uint2* W4 = reinterpret_cast<const uint2*>(W + start);
      for (int64_t j = threadIdx.x; j < nv; j += kThreads) {
        const float4 pv = __ldcs(P4 + j);
        const uint2 wv = __ldcs(W4 + j);
        const int64_t e = start + 4 * j;
        check(pv.x, (uint16_t)(wv.x & 0xffffu), e);
        check(pv.y, (uint16_t)(wv.x >> 16), e + 1);
        check(pv.z, (uint16_t)(wv.y & 0xffffu), e + 2);
        check(pv.w, (uint16_t)(wv.y >> 16), e + 3);
      }
      i0 = start + 4 * nv;
    }
    for (int64_t i = i0 + threadIdx.x; i < stop; i += kThreads) check(P[i], W[i], i);
    if (bad) {
      atomicAdd(out, bad);
      atomicMin(out + 1, key);
    }
  }
}

const void* device_alias(const void* ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return ptr;
  if (a.type == cudaMemoryTypeHost) return a.devicePointer;  // registered / pinned host memory
  return nullptr;  // pageable: not readable by the device
}
}  // namespace

extern "C" int dos_coherence_cuda(const dos_coh_range* ranges, int nranges, int lowp_dtype,
                                  unsigned long long* out, void* stream) {
  if (nranges < 0 || (nranges > 0 && (!ranges || !out))) return dos_set_error(DOS_EINVAL, "bad coherence arguments");
  if (lowp_dtype != DOS_F16 && lowp_dtype != DOS_BF16)
    return dos_set_error(DOS_ETYPE, "working-copy dtype %d unsupported", lowp_dtype);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  for (int base = 0; base < nranges; base += kCohMax) {
    coh_batch b;
    b.n = 0;
    b.lt = lowp_dtype;
    b.base = base;
    b.first[0] = 0;
    for (int j = base; j < nranges && b.n < kCohMax; ++j) {
      const dos_coh_range& r = ranges[j];
      if (r.n < 0 || r.window <= 0 || r.nwin <= 0) return dos_set_error(DOS_EINVAL, "coherence range %d: bad sizes", j);
      const void* p = device_alias(r.p32);
      const void* w = device_alias(r.lowp);
      if (r.n > 0 && (!p || !w))
        return dos_set_error(DOS_EINVAL, "coherence range %d: buffer not device-accessible (pageable host memory?)", j);
      const int i = b.n++;
      b.p[i] = static_cast<const float*>(p);
      b.w[i] = static_cast<const uint16_t*>(w);
      b.len[i] = r.n;
      b.win[i] = r.window < r.n ? r.window : (r.n > 0 ? r.n : 1);
      // whole range: enough contiguous windows to cover it
      const int64_t need = (r.n + b.win[i] - 1) / b.win[i];
      b.nwin[i] = r.n == 0 ? 0 : (r.nwin < need ? r.nwin : need);
      b.first[i + 1] = b.first[i] + b.nwin[i];
    }
    const int64_t pairs = b.first[b.n];
    if (pairs == 0) continue;
    const unsigned grid = (unsigned)(pairs < (int64_t)sm_count() * 8 ? pairs : (int64_t)sm_count() * 8);
    k_coherence<<<grid, kThreads, 0, st>>>(b, out);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return dos_set_error(DOS_ECUDA, "coherence launch failed: %s", cudaGetErrorString(e));
  }
  return DOS_OK;
}

// ---------------------------------------------------------------- shuttle
// The host lane's copy engine for small, LLC-resident staging slots: a
// persistent kernel of a few CTAs, launched at phase start, that serves a
// descriptor queue in mapped pinned host memory (dos_shuttle_ctl).  Host
// threads post descriptors with a few plain stores (no CUDA API call per
// chunk); each descriptor is copied over PCIe (zero-copy loads of the host
// slot) by one CTA, which then publishes done[slot] and, optionally, a flag
// that a stream's cuStreamWaitValue32 is waiting on.
// Because it is a running kernel, no stream's pending wait can ever sit in
// front of its copies (streams share hardware queues; a wait at the head of
// one blocks the others queued behind it — with host threads waiting on
// those copies that deadlocks).
namespace {
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys(const void* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int kShuttleThreads = 512;

// CTA `me` serves descriptors first + me, first + me + G, ... on its own (a
// descriptor is a whole staging slot, copied by the CTA's threads with 4 PCIe
// loads in flight each), so the CTAs never wait for each other.
__global__ void __launch_bounds__(kShuttleThreads) k_shuttle(dos_shuttle_ctl* ctl, uint32_t* flags, uint32_t first) {
  __shared__ uint64_t s_src, s_dst;
  __shared__ uint32_t s_bytes, s_flag_val;
  __shared__ int32_t s_flag_idx;
  __shared__ int s_quit;
  const int tid = threadIdx.x;
  for (uint32_t k = first + blockIdx.x;; k += gridDim.x) {
    const uint32_t slot = k % DOS_SHUTTLE_Q;
    dos_shuttle_desc* d = &ctl->q[slot];
    if (tid == 0) {
      s_quit = 0;
      for (;;) {
        if (ld_acquire_sys(&d->id) == k + 1) break;
        if (ld_acquire_sys(&ctl->stop)) {  // every descriptor is posted before stop: look once more
          if (ld_acquire_sys(&d->id) != k + 1) s_quit = 1;
          break;
        }
        __nanosleep(128);
      }
      if (!s_quit) {
        s_src = ld_relaxed_sys64(&d->src);
        s_dst = ld_relaxed_sys64(&d->dst);
        s_bytes = ld_relaxed_sys(&d->bytes);
        s_flag_idx = (int32_t)ld_relaxed_sys(&d->flag_idx);
        s_flag_val = ld_relaxed_sys(&d->flag_val);
      }
    }
    __syncthreads();
    if (s_quit) return;
    const char* src = reinterpret_cast<const char*>(s_src);
    char* dst = reinterpret_cast<char*>(s_dst);
    const uint32_t bytes = s_bytes;
    if (((s_src | s_dst) & 15u) == 0) {
      const uint32_t units = bytes / 16;
      const uint4* S = reinterpret_cast<const uint4*>(src);
      uint4* D = reinterpret_cast<uint4*>(dst);
      uint32_t u = tid;
      for (; u + 3 * kShuttleThreads < units; u += 4 * kShuttleThreads) {
        const uint4 a = __ldcv(S + u), b = __ldcv(S + u + kShuttleThreads), c = __ldcv(S + u + 2 * kShuttleThreads),
                    e = __ldcv(S + u + 3 * kShuttleThreads);
        D[u] = a;
        D[u + kShuttleThreads] = b;
        D[u + 2 * kShuttleThreads] = c;
        D[u + 3 * kShuttleThreads] = e;
      }
      for (; u < units; u += kShuttleThreads) D[u] = __ldcv(S + u);
      for (uint32_t b = units * 16 + 2 * tid; b < bytes; b += 2 * kShuttleThreads)  // tail (16-bit elements)
        *reinterpret_cast<uint16_t*>(dst + b) = __ldcv(reinterpret_cast<const unsigned short*>(src + b));
    } else {  // unaligned: 16-bit elements
      for (uint32_t e = tid; e < bytes / 2; e += kShuttleThreads)
        reinterpret_cast<uint16_t*>(dst)[e] = __ldcv(reinterpret_cast<const unsigned short*>(src) + e);
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence_system();  // the copy is visible to the host and to every engine
      if (s_flag_idx >= 0) st_release_sys(&flags[s_flag_idx], s_flag_val);
      st_release_sys(&ctl->done[slot], k + 1);
    }
  }
}
}  // namespace

void dos_reserve_sms(int n) { g_reserved_sms.store(n < 0 ? 0 : n, std::memory_order_relaxed); }

int dos_shuttle_launch(dos_shuttle_ctl* ctl_dev, uint32_t* flags_dev, uint32_t first, int nctas, cudaStream_t st) {
  k_shuttle<<<nctas, kShuttleThreads, 0, st>>>(ctl_dev, flags_dev, first);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dos_set_error(DOS_ECUDA, "shuttle launch failed: %s", cudaGetErrorString(e));
  return DOS_OK;
}
