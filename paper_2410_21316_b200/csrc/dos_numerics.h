// dos_numerics.h — per-element arithmetic shared by the sm_100a kernel (K1)
// and the host kernel (H1).  Both tiers must produce the same bits as the
// reference's numba loop (pkg/src/optistate/kernels.py:93-101), so every
// operation is a single IEEE-754 binary32 op with round-to-nearest-even and
// no FMA contraction:
//
//   mi = b1*m + (1-b1)*g ;  vi = b2*v + (1-b2)*(g*g) ;  mh = mi/bc1 ;
//   vh = vi/bc2 ;  p = p - (lr*mh) / (sqrt(vh) + eps)
//
// On the device the ops are spelled with __fmul_rn/__fadd_rn/__fdiv_rn/
// __fsqrt_rn (contraction-proof); the host TUs are compiled with
// -ffp-contract=off -fno-fast-math, where plain operators are exact IEEE.
//
// Half-precision conversions reproduce the reference's rounding:
//   fp32->fp16: numpy astype (core.py:190-198) incl. NaN payload rule
//               (pinned by pkg/tests/test_core.py:31-60,115-123)
//   fp16->fp32: numpy astype (core.py:201-205), exact, payload-preserving
//   fp32->bf16: torch/c10 round_to_nearest_even (NaN -> 0x7FC0)
//   bf16->fp32: exact widening
#pragma once
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define DOS_HD __host__ __device__ __forceinline__
#else
#define DOS_HD static inline __attribute__((always_inline))
#endif

DOS_HD uint32_t dos_fbits(float f) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(f);
#else
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
#endif
}
DOS_HD float dos_bitsf(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}

// IEEE binary32 ops, RNE, never contracted.
#if defined(__CUDA_ARCH__)
#define DOS_MUL(a, b) __fmul_rn((a), (b))
#define DOS_ADD(a, b) __fadd_rn((a), (b))
#define DOS_SUB(a, b) __fsub_rn((a), (b))
#define DOS_DIV(a, b) __fdiv_rn((a), (b))
#define DOS_SQRT(a) __fsqrt_rn((a))
#else
#define DOS_MUL(a, b) ((a) * (b))
#define DOS_ADD(a, b) ((a) + (b))
#define DOS_SUB(a, b) ((a) - (b))
#define DOS_DIV(a, b) ((a) / (b))
#define DOS_SQRT(a) __builtin_sqrtf((a))
#endif

// Scalars of one step, all binary32, prepared once per launch.
struct dos_kscal {
  float lr, b1, b2, eps, bc1, bc2;
  float omb1, omb2;  // 1.0f - b1, 1.0f - b2 as fp32 differences
  float decay;       // 1.0f - lr*wd (AdamW only)
  int adamw;
};

// One element of the update.  Order of operations is the reference's.
DOS_HD void dos_adam_elem(float& p, float& m, float& v, float g, const dos_kscal& s) {
  float pp = p;
  if (s.adamw) pp = DOS_MUL(pp, s.decay);
  const float mi = DOS_ADD(DOS_MUL(s.b1, m), DOS_MUL(s.omb1, g));
  const float vi = DOS_ADD(DOS_MUL(s.b2, v), DOS_MUL(s.omb2, DOS_MUL(g, g)));
  m = mi;
  v = vi;
  const float mh = DOS_DIV(mi, s.bc1);
  const float vh = DOS_DIV(vi, s.bc2);
  p = DOS_SUB(pp, DOS_DIV(DOS_MUL(s.lr, mh), DOS_ADD(DOS_SQRT(vh), s.eps)));
}

// fp32 -> fp16 bits, RNE, overflow -> inf, numpy's NaN rule
// (keep the top 10 payload bits; bump to 0x7C01 if they are all zero).
DOS_HD uint16_t dos_f32_to_f16(float f) {
  uint32_t u = dos_fbits(f);
  const uint32_t sign = (u >> 16) & 0x8000u;
  const uint32_t a = u & 0x7fffffffu;
  uint32_t o;
  if (a > 0x7f800000u) {  // NaN
    o = 0x7c00u + ((a & 0x7fffffu) >> 13);
    o += (o == 0x7c00u) ? 1u : 0u;
  } else if (a >= 0x47800000u) {  // >= 65536 (and inf): overflow
    o = 0x7c00u;
  } else if (a < 0x38800000u) {  // below the smallest fp16 normal 2^-14
    // Adding 0.5 puts the value's 2^-24 quanta in the low mantissa bits
    // with one RNE rounding; subtracting 0.5's bits leaves the subnormal.
    const float t = DOS_ADD(dos_bitsf(a), 0.5f);
    o = dos_fbits(t) - 0x3f000000u;
  } else {  // normal: rebias exponent, round the 13 dropped bits to even
    const uint32_t odd = (a >> 13) & 1u;
    o = (a + 0xc8000fffu + odd) >> 13;  // 0xc8000000 == (15-127)<<23 mod 2^32
  }
  return (uint16_t)(sign | o);
}

// fp16 bits -> fp32, exact (payload and signalling bit preserved like numpy).
DOS_HD float dos_f16_to_f32(uint16_t h) {
  const uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
  const uint32_t e = ((uint32_t)h >> 10) & 0x1fu;
  const uint32_t mant = (uint32_t)h & 0x3ffu;
  uint32_t o;
  if (e == 0x1fu) {
    o = 0x7f800000u | (mant << 13);
  } else if (e == 0u) {
    // subnormal (or zero): mant * 2^-24 is exact in binary32
    o = dos_fbits(DOS_MUL((float)mant, 5.9604644775390625e-8f));
  } else {
    o = ((e + 112u) << 23) | (mant << 13);
  }
  return dos_bitsf(sign | o);
}

// fp32 -> bf16 bits, round-to-nearest-even on the bit pattern (c10 rule).
DOS_HD uint16_t dos_f32_to_bf16(float f) {
  const uint32_t u = dos_fbits(f);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)0x7fc0u;
  return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

DOS_HD float dos_bf16_to_f32(uint16_t b) { return dos_bitsf((uint32_t)b << 16); }
