/* Seeded synthetic scalar fields of the BASELINE configs — the INPUT
 * DEFINITION shared by the device generator (csrc/synth.cu) and every host
 * consumer (the CPU oracle's digests, bench.py's reference arm), so that the
 * GPU and the CPU see identical bytes without shipping volumes around.
 *
 * Not part of the segmentation path. Plain C99, header-only.
 *
 * A Gaussian k = (cx, cy, cz, sigma, amp) is separable:
 *   g_k(x, y, z) = ex_k(x) * ey_k(y) * ez_k(z),  e_k(i) = exp(-(i - c)^2 / (2 sigma^2)).
 * The per-axis factors are tabulated once on the host in float32
 * (plmss_synth_axis_table, a self-contained exp: no libm, no FMA contraction
 * — compile host users with -ffp-contract=off), and every voxel is
 *   s = 0;  for k in order:  w = amp_k * (ey_k(y) * ez_k(z));  s = s + ex_k(x) * w
 * in float32 with every product and sum rounded separately (the device uses
 * __fmul_rn / __fadd_rn), then
 *   f = (float)((double)s + noise * (2u - 1)),  u = (splitmix64(seed ^ v * K) >> 11) * 2^-53
 * in double (u: the reference's (rng() >> 11) * 2^-53 mapping, proj/src/synth.cpp:15-17,
 * over a counter-based hash so any voxel can be generated independently).
 * White noise: f = (float)u. Quantised: t = ((double)f - lo) / (hi - lo),
 * q = floor(t * levels) clamped to [0, levels - 1], lo/hi = min/max of f.
 */
#ifndef PLMSS_SYNTH_H
#define PLMSS_SYNTH_H
#include <stdint.h>

#ifdef __CUDACC__
#define PLMSS_SYNTH_HD __host__ __device__
#else
#define PLMSS_SYNTH_HD
#endif

#ifdef __cplusplus
extern "C" {
#endif

PLMSS_SYNTH_HD static inline uint64_t plmss_synth_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

PLMSS_SYNTH_HD static inline double plmss_synth_uniform01(uint64_t seed, uint64_t v) {
  return (double)(plmss_synth_splitmix64(seed ^ (v * 0xD1B54A32D192ED03ull)) >> 11) * 0x1.0p-53;
}

/* exp(x) for x <= 0 from IEEE +, -, *, / only (Cody-Waite reduction by ln 2,
 * degree-13 Taylor polynomial on |r| <= ln2/2, exact scaling by 2^n); the
 * same bits on every IEEE-754 host. Accurate to a few ulp of double, which
 * is far below the float32 rounding of the tables. */
static inline double plmss_synth_exp(double x) {
  if (x < -740.0) return 0.0;
  if (x > 0.0) x = 0.0;
  const double inv_ln2 = 1.4426950408889634;
  const double ln2_hi = 6.93147180369123816490e-01; /* 32 significant bits: n * ln2_hi is exact */
  const double ln2_lo = 1.90821492927058770002e-10;
  double t = x * inv_ln2;
  int n = (int)(t - 0.5); /* truncation toward zero of t - 0.5: nearest integer for t <= 0 */
  const double r = (x - (double)n * ln2_hi) - (double)n * ln2_lo;
  double p = 1.0 / 6227020800.0; /* 1/13! */
  static const double inv_fact[13] = {1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0,
                                      1.0 / 40320.0,     1.0 / 5040.0,     1.0 / 720.0,     1.0 / 120.0,
                                      1.0 / 24.0,        1.0 / 6.0,        1.0 / 2.0,       1.0,
                                      1.0};
  for (int i = 0; i < 13; ++i) p = p * r + inv_fact[i];
  /* scale by 2^n (n >= -1068 here), exact until the final multiply */
  union {
    double d;
    uint64_t u;
  } s;
  s.u = (uint64_t)(n + 1023) << 52;
  if (n < -1022) {
    /* 2^n is subnormal: multiply in two exact steps */
    p *= 0x1.0p-600;
    s.u = (uint64_t)(n + 600 + 1023) << 52;
  }
  return p * s.d;
}

/* Axis factor table of one Gaussian: out[i] = (float)exp(-(i - c)^2 / (2 sigma^2)), i < len. */
static inline void plmss_synth_axis_table(double c, double sigma, int64_t len, float* out) {
  const double den = 2.0 * sigma * sigma;
  for (int64_t i = 0; i < len; ++i) {
    const double d = (double)i - c;
    out[i] = (float)plmss_synth_exp(-(d * d) / den);
  }
}

#ifdef __cplusplus
}
#endif
#endif
