/* TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * C restatement of the reference's per-element Adam loop
 * (/root/reference/pkg/src/optistate/kernels.py:93-101) and of the
 * working-copy downscale (core.py:190-198, numpy's float16 rounding, written
 * here bit-by-bit after pkg/tests/test_core.py:31-60), compiled with
 * -ffp-contract=off.  Used as the bench's CPU baseline ("port") with all
 * host threads, each thread owning a disjoint contiguous slice (the update
 * is elementwise, so results do not depend on the split).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>

static uint16_t ref_f16_bits(uint32_t f) {
  uint32_t sign = (f >> 16) & 0x8000u, exp = (f >> 23) & 0xffu, sig = f & 0x7fffffu;
  if (exp == 255u) {
    if (sig == 0) return (uint16_t)(sign | 0x7c00u);
    uint32_t out = 0x7c00u + (sig >> 13);
    if (out == 0x7c00u) out += 1;
    return (uint16_t)(sign | out);
  }
  int e = (int)exp - 127 + 15;
  if (e >= 31) return (uint16_t)(sign | 0x7c00u);
  if (e <= 0) {
    if (e < -10) return (uint16_t)sign;
    uint32_t mant = sig | 0x800000u;
    int shift = 14 - e;
    uint32_t out = mant >> shift, dropped = mant & ((1u << shift) - 1u), half = 1u << (shift - 1);
    if (dropped > half || (dropped == half && (out & 1u))) out += 1;
    return (uint16_t)(sign | out);
  }
  uint32_t dropped = sig & 0x1fffu, out = sign | ((uint32_t)e << 10) | (sig >> 13);
  if (dropped > 0x1000u || (dropped == 0x1000u && (out & 1u))) out += 1;
  return (uint16_t)out;
}

static uint16_t ref_bf16_bits(uint32_t u) {
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0u;
  return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

static float ref_f16_to_f32(uint16_t h) {
  uint32_t sign = ((uint32_t)h & 0x8000u) << 16, e = ((uint32_t)h >> 10) & 0x1fu, m = h & 0x3ffu, o;
  if (e == 31u) o = sign | 0x7f800000u | (m << 13);
  else if (e == 0u) {
    float f = ldexpf((float)m, -24);
    memcpy(&o, &f, 4);
    o |= sign;
  } else o = sign | ((e + 112u) << 23) | (m << 13);
  float r;
  memcpy(&r, &o, 4);
  return r;
}

/* lowp: 0 = none, 1 = fp16, 2 = bf16 (same codes as include/dos.h);
 * gkind: 0 = fp32 grads, 1 = fp16 bits, 2 = bf16 bits */
void oracle_adam(float* p, float* m, float* v, const void* g, int gkind, uint16_t* w, int lowp, int64_t n,
                 float lr, float b1, float b2, float eps, float bc1, float bc2) {
  const float one = 1.0f;
  for (int64_t i = 0; i < n; ++i) {
    float gi;
    if (gkind == 0) gi = ((const float*)g)[i];
    else if (gkind == 1) gi = ref_f16_to_f32(((const uint16_t*)g)[i]);
    else {
      uint32_t u = (uint32_t)((const uint16_t*)g)[i] << 16;
      memcpy(&gi, &u, 4);
    }
    float t1 = b1 * m[i];
    float t2 = (one - b1) * gi;
    float mi = t1 + t2;
    float gg = gi * gi;
    float t3 = b2 * v[i];
    float t4 = (one - b2) * gg;
    float vi = t3 + t4;
    m[i] = mi;
    v[i] = vi;
    float mh = mi / bc1;
    float vh = vi / bc2;
    float den = sqrtf(vh) + eps;
    float num = lr * mh;
    float pi = p[i] - num / den;
    p[i] = pi;
    if (lowp) {
      uint32_t u;
      memcpy(&u, &pi, 4);
      w[i] = lowp == 1 ? ref_f16_bits(u) : ref_bf16_bits(u);
    }
  }
}

typedef struct {
  float *p, *m, *v;
  const char* g;
  int gkind;
  uint16_t* w;
  int lowp;
  int64_t lo, hi;
  float lr, b1, b2, eps, bc1, bc2;
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  int gb = j->gkind == 0 ? 4 : 2;
  oracle_adam(j->p + j->lo, j->m + j->lo, j->v + j->lo, j->g + gb * j->lo, j->gkind, j->w ? j->w + j->lo : 0,
              j->lowp, j->hi - j->lo, j->lr, j->b1, j->b2, j->eps, j->bc1, j->bc2);
  return 0;
}

/* Threaded driver: nthreads disjoint slices. */
int oracle_adam_mt(float* p, float* m, float* v, const void* g, int gkind, uint16_t* w, int lowp, int64_t n,
                   float lr, float b1, float b2, float eps, float bc1, float bc2, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  job_t jobs[256];
  int64_t per = (n + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    int64_t lo = per * t < n ? per * t : n, hi = lo + per < n ? lo + per : n;
    job_t j = {p, m, v, (const char*)g, gkind, w, lowp, lo, hi, lr, b1, b2, eps, bc1, bc2};
    jobs[t] = j;
    if (t > 0 && pthread_create(&th[t], 0, run_job, &jobs[t]) != 0) return -1;
  }
  run_job(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], 0);
  return 0;
}
