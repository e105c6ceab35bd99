// chol8.cuh -- the 8x8 corner-covariance factor of the leaf pass.
//
// From a cell posterior [mu (8) | Sigma packed lower (36), corner order c = c0 +
// 2 c1 + 4 c2] to the MC operands [mu_pi (8 double) | L' (36 float)] with
// L = chol(Sigma[pi][pi]) in the corner order pi = (0,3,5,6,1,2,4,7) (R13b) and the
// PSD pivot clamp of R14 (pivot <= 1e-12 max diag -> column zeroed; never fails),
// L' = FOLD_SCALE L (Box-Muller constant folded in, pmc.cu).  FP64 throughout.
#pragma once
#include "common.cuh"

namespace lcp {

// -sqrt(2 ln 2): the Box-Muller factor R = sqrt(-2 ln 2 lg2 u) and its sign
constexpr double FOLD_SCALE = -1.1774100225154747;

// packed index of Sigma[pi(i)][pi(j)], i >= j, in the natural-order packing
__host__ __device__ constexpr int pi8(int i) { return i == 0 ? 0 : i == 1 ? 3 : i == 2 ? 5 : i == 3 ? 6 : i == 4 ? 1 : i == 5 ? 2 : i == 6 ? 4 : 7; }
__host__ __device__ constexpr int pidx(int i, int j) {
  return pi8(i) > pi8(j) ? pi8(i) * (pi8(i) + 1) / 2 + pi8(j) : pi8(j) * (pi8(j) + 1) / 2 + pi8(i);
}

// column J of the left-looking Cholesky, fully unrolled by template recursion
// (a runtime-indexed loop nest would put S and L in local memory)
template <int J>
__device__ __forceinline__ void chol8_col(const double (&S)[36], double (&L)[36], double tol) {
  if constexpr (J < 8) {
    double s = S[J * (J + 3) / 2];
#pragma unroll
    for (int p = 0; p < J; ++p) s -= L[J * (J + 1) / 2 + p] * L[J * (J + 1) / 2 + p];
    const bool live = s > tol;
    const double ljj = live ? sqrt(s) : 0.0;
    const double inv = live ? 1.0 / ljj : 0.0;
    L[J * (J + 3) / 2] = ljj;
#pragma unroll
    for (int i = J + 1; i < 8; ++i) {
      double t = S[i * (i + 1) / 2 + J];
#pragma unroll
      for (int p = 0; p < J; ++p) t -= L[i * (i + 1) / 2 + p] * L[J * (J + 1) / 2 + p];
      L[i * (i + 1) / 2 + J] = live ? t * inv : 0.0;
    }
    chol8_col<J + 1>(S, L, tol);
  }
}

// in: mu[8], sig[36] (natural order); out: mu_out[8] (pi order), L_out[36] (float, FOLD_SCALE L)
__device__ __forceinline__ void chol8_factor(const double (&mu)[8], const double (&sig)[36], double (&mu_out)[8],
                                             float (&L_out)[36]) {
  double S[36];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) S[i * (i + 1) / 2 + j] = sig[pidx(i, j)];
  double md = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) md = fmax(md, S[c * (c + 3) / 2]);
  const double tol = 1e-12 * md;
  double L[36];
  chol8_col<0>(S, L, tol);
  double m2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) m2[i] = mu[pi8(i)];
#pragma unroll
  for (int i = 0; i < 8; ++i) mu_out[i] = m2[i];
#pragma unroll
  for (int p = 0; p < 36; ++p) L_out[p] = (float)(FOLD_SCALE * L[p]);
}

// MC record of a cell: 208 bytes, 16-byte aligned
struct CellRec {
  double mu[8];    // mu_pi
  float L[36];     // FOLD_SCALE chol(Sigma_pi pi), packed row-major lower
};
static_assert(sizeof(CellRec) == 208, "CellRec layout");

}  // namespace lcp
