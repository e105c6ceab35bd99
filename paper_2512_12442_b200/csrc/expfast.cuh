// expfast.cuh -- FP64 e^{-x} and sqrt for the brick kernels' covariance evaluations
// (brick.cu), shared with tools/probes/exp_tab_probe.cu which measures their accuracy.
#pragma once
#include <cuda_runtime.h>

namespace lcp {

// Fast e^{-x} (x >= 0) for the brick's kernel evaluations: n = round(-x log2 e) by
// the 1.5 2^52 magic add, f = -x - n ln2 (Cody-Waite, |f| <= ln2 / 2), e^f by its
// degree-12 Taylor polynomial (truncation < 2e-16 relative), times 2^n built from the
// exponent bits; 0 below 2^-1022.  The coefficients live in the constant bank, so
// every Horner step is one DFMA with a c[] operand (the libm exp materialises each
// 64-bit coefficient with two UMOVs per call).
__constant__ double c_exp_taylor[13] = {
    0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-3,
    0x1.5555555555555p-5, 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
    0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26,
    0x1.1eed8eff8d898p-29};
__constant__ double c_exp_consts[4] = {1.4426950408889634074, 6755399441055744.0, 0x1.62e42fefa39efp-1,
                                       0x1.abc9e3b39803fp-56};

__device__ __forceinline__ double exp_neg_fast(double x) {
  const double t = fma(-x, c_exp_consts[0], c_exp_consts[1]);
  const double n = t - c_exp_consts[1];
  double f = fma(n, -c_exp_consts[2], -x);
  f = fma(n, -c_exp_consts[3], f);
  double p = c_exp_taylor[12];
#pragma unroll
  for (int i = 11; i >= 0; --i) p = fma(p, f, c_exp_taylor[i]);
  const int ni = __double2loint(t);
  const double scale = __hiloint2double((ni + 1023) << 20, 0);
  return (ni < -1022 || x > 745.0) ? 0.0 : p * scale;   // x > 745: also guards the magic-add range
}

// Table-driven e^{-x} (x >= 0) for the brick's kernel evaluations: n = round(-64 x log2 e)
// by the magic add, g = -x - n ln2/64 (Cody-Waite inside two FMAs, |g| <= ln2/128), e^g by
// its degree-5 Taylor polynomial (truncation < 4e-17 relative), times 2^(j/64) from a
// 64-entry shared-memory table (j = n mod 64) and 2^floor(n/64) from the exponent bits.
// 11 FP64 operations and a 5-deep Horner chain instead of exp_neg_fast's 17 and 12.
__constant__ double c_exp2_64[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0};
__constant__ double c_exp_tab_consts[4] = {92.332482616893656877, 6755399441055744.0,
                                           0x1.62e42fefa39efp-7, 0x1.abc9e3b39803fp-62};

__device__ __forceinline__ double exp_neg_tab(double x, const double* __restrict__ tab) {
  const double t = fma(-x, c_exp_tab_consts[0], c_exp_tab_consts[1]);
  const double n = t - c_exp_tab_consts[1];
  double gg = fma(n, -c_exp_tab_consts[2], -x);
  gg = fma(n, -c_exp_tab_consts[3], gg);
  double p = fma(gg, 0x1.1111111111111p-7, 0x1.5555555555555p-5);
  p = fma(p, gg, 0x1.5555555555555p-3);
  p = fma(p, gg, 0.5);
  p = fma(p, gg, 1.0);
  p = fma(p, gg, 1.0);
  const int ni = __double2loint(t);
  const int m = ni >> 6;
  const double scale = __hiloint2double((m + 1023) << 20, 0);
  return (m < -1022 || x > 745.0) ? 0.0 : (tab[ni & 63] * p) * scale;
}

// exp_neg_tab without branches (k_brick's phase 1): x clamped to 745 (e^-745 is below the
// smallest subnormal), 2^m applied as 2^(m >> 1) 2^(m - (m >> 1)) so that m < -1022 gives
// the subnormal (or zero) product instead of a branch to 0; identical to exp_neg_tab
// whenever that one returns a normal number.  The degree-3..5 Taylor coefficients come
// from the constant bank (DFMA c[] operands instead of UMOV pairs).
__constant__ double c_exp_tab_poly[3] = {0x1.1111111111111p-7, 0x1.5555555555555p-5, 0x1.5555555555555p-3};

__device__ __forceinline__ double exp_neg_tab_bf(double x, const double* __restrict__ tab) {
  x = x < 745.0 ? x : 745.0;
  const double t = fma(-x, c_exp_tab_consts[0], c_exp_tab_consts[1]);
  const double n = t - c_exp_tab_consts[1];
  double gg = fma(n, -c_exp_tab_consts[2], -x);
  gg = fma(n, -c_exp_tab_consts[3], gg);
  double p = fma(gg, c_exp_tab_poly[0], c_exp_tab_poly[1]);
  p = fma(p, gg, c_exp_tab_poly[2]);
  p = fma(p, gg, 0.5);
  p = fma(p, gg, 1.0);
  p = fma(p, gg, 1.0);
  const int ni = __double2loint(t);
  const int m = ni >> 6, m1 = m >> 1, m2 = m - m1;
  const double s1 = __hiloint2double((m1 + 1023) << 20, 0), s2 = __hiloint2double((m2 + 1023) << 20, 0);
  return ((tab[ni & 63] * p) * s1) * s2;
}

// sqrt of x > 0 (no zero select: callers pass r^2 + 1e-300, which equals r^2 for every
// r^2 above ~1e-284 and keeps rsqrt finite at r = 0).  One Newton step on the MUFU.RSQ64H
// seed plus the final correction is already correctly rounded (0 ulp from __dsqrt_rn on
// 6.7e7 log-uniform values in [1e-12, 1e12], tools/probes/sqrt_probe.cu; without the
// Newton step 11 522 ulp)
__device__ __forceinline__ double sqrt_pos(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-0.5 * x, y * y, 1.5);
  const double r = x * y;
  return fma(0.5 * y, fma(-r, r, x), r);
}

// branch-free sqrt: MUFU.RSQ64H seed, two Newton steps on 1/sqrt, one on sqrt (~1 ulp);
// sqrt(0) = 0 by a select (libm sqrt branches to a slow path per element)
__device__ __forceinline__ double sqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-0.5 * x, y * y, 1.5);
  y = y * fma(-0.5 * x, y * y, 1.5);
  double r = x * y;
  r = fma(0.5 * y, fma(-r, r, x), r);
  return x > 0.0 ? r : 0.0;
}

}  // namespace lcp
