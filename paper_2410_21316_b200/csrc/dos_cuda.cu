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

#include "dos_internal.h"
#include "dos_numerics.h"

namespace {

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

// Vector body over [base, base + 8*nvec), plus `nscalar` scalar elements
// (the unaligned head [0, head) and the tail after the vector body).
template <int GT, int LT>
__global__ void __launch_bounds__(kThreads)
    k_adam(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
           const void* __restrict__ g, void* __restrict__ lp, int64_t head, int64_t nvec,
           int64_t n, dos_kscal s) {
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
    load_g8(gv, GT, i, gg);
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
      __stcs(reinterpret_cast<uint4*>(lv) + i, make_uint4(w[0], w[1], w[2], w[3]));
    }
  }

  // scalar head + tail
  const int64_t vec_end = head + kVec * nvec;
  const int64_t nscalar = head + (n - vec_end);
  for (int64_t j = tid; j < nscalar; j += nthr) {
    const int64_t e = j < head ? j : vec_end + (j - head);
    float pe = p[e], me = m[e], ve = v[e];
    dos_adam_elem(pe, me, ve, load_g1(g, GT, e), s);
    p[e] = pe;
    m[e] = me;
    v[e] = ve;
    if (LT != DOS_NONE) reinterpret_cast<uint16_t*>(lp)[e] = to_lowp(pe, LT);
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
                 int64_t n, const dos_kscal& s, cudaStream_t st) {
  const int64_t work = nvec > 0 ? nvec : n;
  k_adam<GT, LT><<<grid_for(work), kThreads, 0, st>>>(p, m, v, g, lp, head, nvec, n, s);
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

int dos_adam_launch(float* p, float* m, float* v, const void* g, int gt, void* lp, int lt, int64_t n,
                    const dos_kscal& s, cudaStream_t st) {
  if (n == 0) return DOS_OK;
  const void* ptrs[5] = {p, m, v, g, lp};
  const int eb[5] = {4, 4, 4, gt == DOS_F32 ? 4 : 2, 2};
  int64_t head = common_head(ptrs, eb, lt == DOS_NONE ? 4 : 5, n);
  int64_t nvec = 0;
  if (head < 0) {
    head = n;  // no common alignment: everything takes the scalar path
  } else {
    nvec = (n - head) / kVec;
  }
#define DOS_CASE(G, L) \
  if (gt == G && lt == L) { launch_adam<G, L>(p, m, v, g, lp, head, nvec, n, s, st); }
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
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dos_set_error(DOS_ECUDA, "upscale launch failed: %s", cudaGetErrorString(e));
  return DOS_OK;
}
