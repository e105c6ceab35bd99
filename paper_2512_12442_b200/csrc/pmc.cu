// pmc.cu -- lcp_pmc_cells: SURVEY §8(a) rows a7-a9.
//
//  a7  cell posterior (marginals.cu: k_cell_posterior), cells grouped by bucket
//  a8  k_chol8 : 8x8 Cholesky of Sigma in FP64 with the PSD pivot clamp (R14)
//      k_pmc   : warp per cell; lane l draws samples s = l, l+32, ...:
//                Philox4x32-10, key = seed, counter (cell lo, iso, cell hi, w) (R13):
//                z0..z3 from three words of the lane group's stream (w = 2 (3g + j),
//                R13c), z4..z7 from w = 2s + 1; uniforms from the low 23 bits
//                (and the top bytes); Box-Muller; y = mu +
//                L z in FP32; crossing = not all y < th and not all y > th
//                (R5, R24).  LCP = count / N.
//  a9  k_scatter : dense field, zero off the leaves.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "chol8.cuh"
#include "ctx.h"

namespace lcp {

#ifndef PMC_SCALAR_LZ   // 1: scalar FFMA chains for the phase-1 L'z instead of FFMA2
#define PMC_SCALAR_LZ 0
#endif
#ifndef PMC_ABS_LG2
#define PMC_ABS_LG2 1
#endif

// The constant -sqrt(2 ln 2) of Box-Muller's R = sqrt(-2 ln 2 lg2(u_a)) (and its sign)
// is carried by L' (chol8.cuh stores FOLD_SCALE L), so k_pmc draws z / FOLD_SCALE.
constexpr int64_t PMC_CHUNK = (int64_t)1 << 23;   // cells per posterior/MC chunk (2.9 GB of records)

__global__ void k_cell_bucket(Geom g, const int64_t* __restrict__ cells, int64_t n, int32_t* __restrict__ bkt,
                              int* __restrict__ derr) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  int64_t cell = cells[q];
  int64_t ncell = (int64_t)g.cells[0] * g.cells[1] * g.cells[2];
  if (cell < 0 || cell >= ncell) {
    atomicOr(derr, DERR_OVERFLOW);
    cell = 0;
  }
  bkt[q] = cell_bucket(g, cell);
}

// number of positions where the bucket changes (runs - 1)
__global__ void k_count_runs(const int32_t* __restrict__ bkt, int64_t n, unsigned long long* __restrict__ out) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned v = (q + 1 < n && bkt[q] != bkt[q + 1]) ? 1u : 0u;
  unsigned b = __ballot_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(out, (unsigned long long)__popc(b));
}

__global__ void k_gather_bkt(const int32_t* __restrict__ bkt, const int64_t* __restrict__ perm, int64_t n,
                             int32_t* __restrict__ out) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) out[q] = bkt[perm[q]];
}

// a8: in-place: rec = [mu (8 double) | Sigma packed (36 double)] ->
//                     [mu_pi (8 double) | L' packed row-major lower (36 float) | unused]
// (chol8.cuh).  The tetrahedral corner order makes the last four corners' conditional
// spread small given the first four (used by the exact early decision of k_pmc).
__global__ void k_chol8(double* __restrict__ post, int64_t n) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  double* rec = post + 44 * q;
  double mu[8], sig[36], mo[8];
  float Lf[36];
#pragma unroll
  for (int i = 0; i < 8; ++i) mu[i] = rec[i];
#pragma unroll
  for (int p = 0; p < 36; ++p) sig[p] = rec[8 + p];
  chol8_factor(mu, sig, mo, Lf);
#pragma unroll
  for (int i = 0; i < 8; ++i) rec[i] = mo[i];
  float4* L4 = reinterpret_cast<float4*>(rec + 8);
#pragma unroll
  for (int t = 0; t < 9; ++t) L4[t] = make_float4(Lf[4 * t], Lf[4 * t + 1], Lf[4 * t + 2], Lf[4 * t + 3]);
}

// refine-time brick pass output (44-double slots, 64 per brick unit) -> MC records
// indexed by the cell's Morton code in the virtual 2^Lfull cube.  CTA per brick: the
// brick's 64 slots are staged through shared memory (row stride 45 doubles: conflict-free)
// so that both the 22.5 KB read and the 13 KB record write (the brick's 64 cells are 64
// consecutive Morton codes) are coalesced.  Records of out-of-grid cells of a clipped brick
// get written too; no leaf list ever names them.
constexpr int REC_STR = 45;
__global__ void __launch_bounds__(64) k_chol8_rec(Geom g, const uint64_t* __restrict__ bricks, int64_t nb,
                                                  const uint8_t* __restrict__ ucomp, const double* __restrict__ post,
                                                  CellRec* __restrict__ recs) {
  __shared__ __align__(16) double sbuf[64 * REC_STR];
  const int64_t u = blockIdx.x;
  if (u >= nb || !ucomp[u]) return;   // brick done by an earlier refine: its records stand
  const int q = threadIdx.x;
  const double* src = post + 64 * 44 * u;
  for (int e = q; e < 64 * 44; e += 64) sbuf[(e / 44) * REC_STR + e % 44] = src[e];
  __syncthreads();
  double mu[8], sig[36];
#pragma unroll
  for (int i = 0; i < 8; ++i) mu[i] = sbuf[q * REC_STR + i];
#pragma unroll
  for (int p = 0; p < 36; ++p) sig[p] = sbuf[q * REC_STR + 8 + p];
  double mo[8];
  float Lf[36];
  chol8_factor(mu, sig, mo, Lf);
  __syncthreads();   // staging buffer becomes the output buffer: 64 records by local Morton code
  CellRec* so = reinterpret_cast<CellRec*>(sbuf);
  CellRec& r = so[morton3(q & 3, (q >> 2) & 3, q >> 4)];
#pragma unroll
  for (int i = 0; i < 8; ++i) r.mu[i] = mo[i];
#pragma unroll
  for (int p = 0; p < 36; ++p) r.L[p] = Lf[p];
  __syncthreads();
  int bi, bj, bk;
  node_unkey(bricks[u], bi, bj, bk);
  float4* dst = reinterpret_cast<float4*>(recs + rec_index(g, 4 * bi, 4 * bj, 4 * bk));
  const float4* s4 = reinterpret_cast<const float4*>(sbuf);
  for (int e = q; e < 64 * (int)(sizeof(CellRec) / 16); e += 64) dst[e] = s4[e];
}

// The same conversion without shared-memory staging, thread per cell (one-warp CTAs, two per
// brick): each thread reads its own 352-B slot with 16-B loads and writes its 208-B record with
// 16-B stores.  0.92 ms per 131 072-brick chunk against 1.13 ms for the staged kernel above
// (CHOL8_REC_DIRECT = 0).  Run beside the next chunk's k_brick on a second stream it would slow
// k_brick by more than it hides (c5 pass 386.7 -> 396.8 ms with a matching carve-out; without
// one the two never share an SM).  Records bit-identical.
#ifndef CHOL8_REC_DIRECT
#define CHOL8_REC_DIRECT 1
#endif
__global__ void __launch_bounds__(32) k_chol8_rec_direct(Geom g, const uint64_t* __restrict__ bricks, int64_t nb,
                                                         const uint8_t* __restrict__ ucomp,
                                                         const double* __restrict__ post, CellRec* __restrict__ recs) {
  const int64_t u = blockIdx.x >> 1;
  if (u >= nb || !ucomp[u]) return;   // brick done by an earlier refine: its records stand
  const int q = ((blockIdx.x & 1) << 5) | threadIdx.x;   // local cell of the brick (x fastest)
  const double2* src = reinterpret_cast<const double2*>(post + 44 * (64 * u + q));
  double mu[8], sig[36];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const double2 v = src[t];
    mu[2 * t] = v.x;
    mu[2 * t + 1] = v.y;
  }
#pragma unroll
  for (int t = 0; t < 18; ++t) {
    const double2 v = src[4 + t];
    sig[2 * t] = v.x;
    sig[2 * t + 1] = v.y;
  }
  double mo[8];
  float Lf[36];
  chol8_factor(mu, sig, mo, Lf);
  int bi, bj, bk;
  node_unkey(bricks[u], bi, bj, bk);
  CellRec* r = recs + rec_index(g, 4 * bi, 4 * bj, 4 * bk) + morton3(q & 3, (q >> 2) & 3, q >> 4);
  double2* m2 = reinterpret_cast<double2*>(r->mu);
#pragma unroll
  for (int t = 0; t < 4; ++t) m2[t] = make_double2(mo[2 * t], mo[2 * t + 1]);
  float4* l4 = reinterpret_cast<float4*>(r->L);
#pragma unroll
  for (int t = 0; t < 9; ++t) l4[t] = make_float4(Lf[4 * t], Lf[4 * t + 1], Lf[4 * t + 2], Lf[4 * t + 3]);
}

cudaError_t launch_chol8_rec(Ctx& c, const uint64_t* bricks, int64_t nb, const double* post) {
  if (nb <= 0) return cudaSuccess;
  if (CHOL8_REC_DIRECT)
    k_chol8_rec_direct<<<(unsigned)(2 * nb), 32, 0, c.stream>>>(c.g, bricks, nb, c.brick_unit.as<uint8_t>(), post,
                                                                 c.crec.as<CellRec>());
  else
    k_chol8_rec<<<(unsigned)nb, 64, 0, c.stream>>>(c.g, bricks, nb, c.brick_unit.as<uint8_t>(), post,
                                                   c.crec.as<CellRec>());
  ++c.n_launch;
  return cudaGetLastError();
}

// 1 in cov[0] if some cell's brick has no record (the list needs the posterior path)
__global__ void k_cells_covered(Geom g, const int64_t* __restrict__ cells, int64_t n,
                                const uint8_t* __restrict__ bdone, unsigned long long* __restrict__ cov) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool miss = false;
  if (q < n) {
    const int64_t cell = cells[q];
    if (cell < 0 || cell >= (int64_t)g.cells[0] * g.cells[1] * g.cells[2]) {
      miss = true;   // invalid id: take the posterior path, which reports it
    } else {
      int i, j, k;
      cell_ijk(g, cell, i, j, k);
      miss = !rec_in_slab(g, k) || !bdone[rec_index(g, i, j, k) >> 6];
    }
  }
  if (__any_sync(0xffffffffu, miss) && (threadIdx.x & 31) == 0) atomicOr(cov, 1ull);
}

// Philox4x32-10 round keys (k0 + r W0, k1 + r W1), r = 0..9, passed as a kernel
// parameter so that every XOR takes its key straight from the constant bank.
struct PhiloxKeys {
  uint32_t k[20];
};

__device__ __forceinline__ void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                              const PhiloxKeys& K, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                              uint32_t& r3) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ K.k[2 * i];
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ K.k[2 * i + 1];
    c0 = n0;
    c1 = (uint32_t)p1;
    c2 = n2;
    c3 = (uint32_t)p0;
  }
  r0 = c0; r1 = c1; r2 = c2; r3 = c3;
}

// 1.0f | (r mod 2^23) as one LOP3 (r & 0x7fffff) | one, `one` = 0x3f800000 held in a
// register (with two immediates ptxas would emit two LOP3)
#ifndef PMC_LOP_MERGE
#define PMC_LOP_MERGE 1
#endif
__device__ __forceinline__ uint32_t mant1(uint32_t r, uint32_t one) {
#if PMC_LOP_MERGE
  uint32_t d;
  asm("lop3.b32 %0, %1, 0x7fffff, %2, 0xEA;" : "=r"(d) : "r"(r), "r"(one));
  return d;
#else
  return 0x3f800000u | (r & 0x7fffffu);
#endif
}
// u = (r mod 2^23 + 1/2) 2^-23, exact: one LOP3 + one FADD
__device__ __forceinline__ float u23(uint32_t r, uint32_t one) {
  return __uint_as_float(mant1(r, one)) - (1.0f - 0x1p-24f);
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// u >= 2^-24 is a normal number: no denormal fix-up needed (MUFU.LG2 alone)
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Box-Muller (R13) with the scale folded into L' (chol8.cuh stores FOLD_SCALE L): returns
// (z0, z1) / FOLD_SCALE = (r cos 2 pi ub, r sin 2 pi ub), r = sqrt(-lg2 ua) = R / sqrt(2 ln 2).
// The angle is taken in (-pi, pi) as 2 pi (ub - 1/2), which flips both signs (absorbed by
// FOLD_SCALE < 0); with F = 1 + (r mod 2^23) 2^-23 it is one FFMA: 2 pi F - 2 pi (3/2 - 2^-24).
// Packed FP32x2 arithmetic (sm_100a FFMA2 / FMUL2): two lanes of FP32 per
// instruction, each rounded exactly as the scalar fmaf / multiply; a pair built
// from one scalar twice is issued as a broadcast operand.
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk(float a, float b) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(f2_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2_t ffma2(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2_t fmul2(f2_t a, f2_t b) {
  f2_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// Box-Muller with the two products r cos, r sin in one FMUL2: returns pk(z0, z1)
__device__ __forceinline__ f2_t box_muller2(uint32_t ra, uint32_t rb, uint32_t one) {
  float ua = u23(ra, one);
  float fb = __uint_as_float(mant1(rb, one));
#if PMC_ABS_LG2
  // |lg2 u| (u < 1, so -lg2 u except where the approximation strays above 0 by ~2^-22):
  // the absolute value is a free MUFU operand modifier, where max(-lg2 u, 0) costs an FMNMX
  float r = sqrt_approx(fabsf(lg2_approx(ua)));
#else
  float r = sqrt_approx(fmaxf(-lg2_approx(ua), 0.0f));
#endif
  float s, co;
  __sincosf(fmaf(6.283185307179586f, fb, -9.424777586727f), &s, &co);
  return fmul2(pk(co, s), pk(r, r));
}

// Largest |z| Box-Muller can produce: u_a >= 2^-24 gives R <= sqrt(48 ln 2) = 5.7668;
// 5.7684 adds the lg2/sqrt approximation error.
constexpr float ZMAX = 5.7684f;
// one warp (one cell) per CTA: a CTA's resources are released when its own cell is done,
// so cells with more phase-2 work do not hold idle warps of their CTA (8-warp CTAs: 99.9 ms
// per 4.19 M-cell chunk; 1-warp CTAs: 97.0 ms with a 128-register bound, 95.7 ms with the
// looser bound below -- the same 118 registers, 17 warps per SM, a better schedule)
#ifndef PMC_WARPS
#define PMC_WARPS 1
#endif
#ifndef PMC_ILP   // 2: two samples per lane in flight (T <= 4); 1: one (T > 4 always)
#define PMC_ILP 2
#endif
constexpr int QCAP = 96;            // pending samples per warp (< 32 + 2 pushes of 32)
constexpr int QROWS = QCAP + 32;    // + a trash row per lane: queue stores are branch-free

// k_pmc<T>: exact two-phase evaluation of the PMC count for
// T isovalues at once (T = 1: the single-isovalue pass; T > 1: NEXT-3, R27).
// Corner values are taken relative to the first isovalue, m_c = mu_c - th_0
// (FP64 difference rounded once); isovalue t is the offset dl_t = th_t - th_0
// (dl_0 = 0), and a sample crosses t iff min_c y_c <= dl_t <= max_c y_c.
// Phase 1 takes the sample's three words of its lane group's phase-1 word stream
// (normals z0..z3, R13c: three Philox blocks serve four samples) and forms
// y_c exactly for the first four corners and y_c - R_c for the other four,
// where |R_c| = |sum_{d>=4} L_cd z_d| <= B_c = ZMAX sum_{d>=4} |L_cd| (+ rounding
// slack).  That brackets max_c y_c in [LMX, UMX] and min_c y_c in [LMN, UMN].
// If for every isovalue the bounds fix the outcome (dl > UMX or dl < LMN: no
// crossing; UMN <= dl <= LMX: crossing) the sample is counted; otherwise it is
// queued in shared memory and, 32 at a time, phase 2 draws the second Philox
// block (z4..z7), finishes the sample and counts every isovalue exactly.  Every
// sample is decided exactly as the one-pass FP32 evaluation decides it; the
// count is the same estimator.
// register bound: at least PMC_MINBLOCKS one-warp CTAs per SM for T <= 8 (70 registers, 28 warps;
// with R13c's packed words: 79.0 ms per c5 chunk against 81.3 at 94 registers and 79.9 at 80),
// 8 for T = 12, 16 (whose isovalue counters would spill at 70)
#ifndef PMC_MINBLOCKS
#define PMC_MINBLOCKS 26
#endif
#ifndef PMC_QUEUE_PRED
#define PMC_QUEUE_PRED 0
#endif
#ifndef PMC_UNIFORM_Q
#define PMC_UNIFORM_Q 1
#endif
constexpr int MAX_ISO = 16;
struct IsoOffsets {
  float dl[MAX_ISO];   // th_t - th_0 (padding: +inf, never crosses)
  int n_out;           // isovalues written (T is padded up to an instantiated size)
  uint32_t one_bits;   // 0x3f800000 (the bits of 1.0f)
};

template <int T>
__global__ void __launch_bounds__(PMC_WARPS * 32, (T <= 8 ? PMC_MINBLOCKS : 8))
    k_pmc(const Geom g, const int64_t* __restrict__ cells, const double* __restrict__ post, int64_t rec_stride,
          int rec_by_morton,
          int64_t n, double theta, const IsoOffsets D, uint32_t N, const PhiloxKeys K, uint32_t iso, const uint32_t* __restrict__ mask,
          int64_t out_stride, float* __restrict__ out, unsigned long long* __restrict__ n_phase2) {
  constexpr int ILP = (T <= 4) ? PMC_ILP : 1;
  // queue, slot-major: (lo4..lo7), (max y0..3, min y0..3, s, -)
  __shared__ float4 sq[PMC_WARPS][2][QROWS];   // SoA: 16-B stores of consecutive slots are contiguous
  __shared__ unsigned int s_p2;
  if (threadIdx.x == 0) s_p2 = 0;
  __syncthreads();
  // one-warp CTAs: the cell index is blockIdx.x, provably warp-uniform, so ptxas keeps the
  // Philox round keys and other per-cell scalars in uniform registers (118 -> 94 registers)
  const int64_t q = (PMC_WARPS == 1 && PMC_UNIFORM_Q) ? (int64_t)blockIdx.x : (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool live = q < n;
  // m[c] = mu_c - th_0 (c < 4); mB[c] = mu_c - th_0 - B_c for the last four corners
  float m[4], mB[4], L[36], B[4];
  uint32_t c1 = 0, c2 = 0;
  constexpr float ZB = (float)(ZMAX / 1.1774100225154747);   // bound on |z / FOLD_SCALE|
  if (live) {
    const int64_t cell = cells[q];
    c1 = (uint32_t)(uint64_t)cell;
    c2 = (uint32_t)((uint64_t)cell >> 32);
    int64_t ri = q;
    if (rec_by_morton) {
      int ci, cj, ck;
      cell_ijk(g, cell, ci, cj, ck);
      ri = rec_index(g, ci, cj, ck);
    }
    const double* rec = post + rec_stride * ri;
    float mm[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) mm[c] = (float)(rec[c] - theta);
    const float4* L4 = reinterpret_cast<const float4*>(rec + 8);
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      float4 v = L4[t];
      L[4 * t] = v.x; L[4 * t + 1] = v.y; L[4 * t + 2] = v.z; L[4 * t + 3] = v.w;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) m[c] = mm[c];
#pragma unroll
    for (int c = 4; c < 8; ++c) {
      float all = fabsf(mm[c]);
#pragma unroll
      for (int d = 0; d <= c; ++d) all += ZB * fabsf(L[c * (c + 1) / 2 + d]);
      // z4, z5 (and z6, z7) are one Box-Muller pair r (cos, sin) with r <= ZB, so
      // |L'_c4 z4 + L'_c5 z5| <= ZB ||(L'_c4, L'_c5)||_2 (same for 6, 7): the tail is
      // bounded by ZB (||.|| + ||.||); the slack covers the sin/cos approximation
      // and the FP32 rounding of the partial sums, so phase-1 decisions equal the
      // one-pass FP32 decisions
      const float l4 = L[c * (c + 1) / 2 + 4];
      const float l5 = c >= 5 ? L[c * (c + 1) / 2 + 5] : 0.0f;
      const float l6 = c >= 6 ? L[c * (c + 1) / 2 + 6] : 0.0f;
      const float l7 = c >= 7 ? L[c * (c + 1) / 2 + 7] : 0.0f;
      const float tail = sqrtf(l4 * l4 + l5 * l5) + sqrtf(l6 * l6 + l7 * l7);
      B[c - 4] = ZB * tail * (1.0f + 1e-5f) + 1e-6f * all;
      mB[c - 4] = mm[c] - B[c - 4];
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) m[c] = mB[c] = B[c] = 0.0f;
#pragma unroll
    for (int p = 0; p < 36; ++p) L[p] = 0.0f;
  }
  // isovalue offsets: literal 0 for the first (single-isovalue code = T == 1)
  auto dl = [&](int t) -> float { return t == 0 ? 0.0f : D.dl[t]; };
  const uint32_t Nl = live ? N : 0u;
  uint32_t cnt[T];
#pragma unroll
  for (int t = 0; t < T; ++t) cnt[t] = 0;
  int qn = 0;   // warp-uniform queue length
  unsigned p2 = 0;
  float4* qv = &sq[wid][0][0];
  float4* qw = &sq[wid][1][0];
  // L' as FFMA2 operands: corner pairs (0,1) (2,3) (4,5) (6,7) per normal d
  f2_t P01 = pk(L[0], L[1]), P23[3], P45[4], P67[4];
#pragma unroll
  for (int d = 0; d < 3; ++d) P23[d] = pk(L[3 + d], L[6 + d]);
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    P45[d] = pk(L[10 + d], L[15 + d]);
    P67[d] = pk(L[21 + d], L[28 + d]);
  }
  const float L11 = L[2], L33 = L[9];
  const f2_t M01 = pk(m[0], m[1]), M23 = pk(m[2], m[3]), MB45 = pk(mB[0], mB[1]), MB67 = pk(mB[2], mB[3]);
  const f2_t B45 = pk(B[0], B[1]), B67 = pk(B[2], B[3]), TWO = pk(2.0f, 2.0f);
  const uint32_t ONE = D.one_bits;   // 0x3f800000 through a kernel parameter: a register, not an immediate
  // phase 1 of sample s: returns true (and the stash) if the sample is undecided.
  // y_c for c < 4 exactly; lo_c = y_c - B_c - R_c and hi_c = lo_c + 2 B_c for c >= 4.
  // Same FP32 operations in the same order as the scalar chains y = fma(L'_cd, z_d, y).
  // phase 1 of sample s from its three words (A, B, C) of the group's word stream (R13c):
  // (z0, z1) = BM(u(A), u(C)), (z2, z3) = BM(u(B), u(A[24..31] | B[24..31] << 8 | C[24..31] << 16))
  // decision and stash of one sample from y (corners 0-3), lo and hi (corners 4-7)
  auto decide = [&](uint32_t s, const float* y, const float* lo, const float* hi, bool valid, float4& st0,
                    float4& st1) -> bool {
    // 3-input chains (FMNMX3)
    const float mx03 = fmaxf(fmaxf(fmaxf(y[0], y[1]), y[2]), y[3]);
    const float mn03 = fminf(fminf(fminf(y[0], y[1]), y[2]), y[3]);
    const float hi_max = fmaxf(fmaxf(fmaxf(fmaxf(mx03, hi[0]), hi[1]), hi[2]), hi[3]);
    const float hi_min = fminf(fminf(fminf(fminf(mn03, hi[0]), hi[1]), hi[2]), hi[3]);
    const float lo_max = fmaxf(fmaxf(fmaxf(fmaxf(mx03, lo[0]), lo[1]), lo[2]), lo[3]);
    const float lo_min = fminf(fminf(fminf(fminf(mn03, lo[0]), lo[1]), lo[2]), lo[3]);
    bool decided = true;
    bool cross[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const float d = dl(t);
      cross[t] = lo_max >= d && hi_min <= d;
      decided = decided && (hi_max < d || lo_min > d || cross[t]);
    }
    if (decided && valid) {
#pragma unroll
      for (int t = 0; t < T; ++t) cnt[t] += cross[t] ? 1u : 0u;
    }
    st0 = make_float4(lo[0], lo[1], lo[2], lo[3]);
    st1 = make_float4(mx03, mn03, __uint_as_float(s), 0.0f);
    return !decided && valid;
  };
  auto phase1w = [&](uint32_t s, uint32_t wa, uint32_t wb, uint32_t wc, bool valid, float4& st0,
                     float4& st1) -> bool {
    const uint32_t wd = __byte_perm(__byte_perm(wa, wb, 0x0073), wc, 0x0710);
    const f2_t zA = box_muller2(wa, wc, ONE), zB = box_muller2(wb, wd, ONE);
    float z[4];
    upk(zA, z[0], z[1]);
    upk(zB, z[2], z[3]);
    float y[4], lo[4], hi[4];
#if PMC_SCALAR_LZ
    // scalar FFMA chains, the same roundings in the same order as the FFMA2 form
    y[0] = fmaf(L[0], z[0], m[0]);
    y[1] = fmaf(L[2], z[1], fmaf(L[1], z[0], m[1]));
    y[2] = m[2];
    y[3] = m[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      y[2] = fmaf(L[3 + d], z[d], y[2]);
      y[3] = fmaf(L[6 + d], z[d], y[3]);
    }
    y[3] = fmaf(L33, z[3], y[3]);
#pragma unroll
    for (int c = 0; c < 4; ++c) lo[c] = mB[c];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      lo[0] = fmaf(L[10 + d], z[d], lo[0]);
      lo[1] = fmaf(L[15 + d], z[d], lo[1]);
      lo[2] = fmaf(L[21 + d], z[d], lo[2]);
      lo[3] = fmaf(L[28 + d], z[d], lo[3]);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) hi[c] = fmaf(2.0f, B[c], lo[c]);
#else
    f2_t A01 = ffma2(P01, pk(z[0], z[0]), M01);
    f2_t A23 = M23, A45 = MB45, A67 = MB67;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const f2_t zd = pk(z[d], z[d]);
      if (d < 3) A23 = ffma2(P23[d], zd, A23);
      A45 = ffma2(P45[d], zd, A45);
      A67 = ffma2(P67[d], zd, A67);
    }
    upk(A01, y[0], y[1]);
    upk(A23, y[2], y[3]);
    y[1] = fmaf(L11, z[1], y[1]);
    y[3] = fmaf(L33, z[3], y[3]);
    upk(A45, lo[0], lo[1]);
    upk(A67, lo[2], lo[3]);
    upk(ffma2(TWO, B45, A45), hi[0], hi[1]);
    upk(ffma2(TWO, B67, A67), hi[2], hi[3]);
#endif
    return decide(s, y, lo, hi, valid, st0, st1);
  };
  // phase-2 operands: columns 4..7 of corners 4..7
  const f2_t Q45[1] = {pk(L[14], L[19])};
  const f2_t Q67[3] = {pk(L[25], L[32]), pk(L[26], L[33]), pk(L[27], L[34])};
  const float L55 = L[20], L77 = L[35];
  // branch-free enqueue of two samples per lane: pending lanes take consecutive
  // slots (all a's, then all b's), the others their trash row
  const unsigned lt = (1u << lane) - 1u;
  auto push2 = [&](bool pa, const float4& a0, const float4& a1, bool pb, const float4& b0, const float4& b1) {
    unsigned ma, mb;
    asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; vote.sync.ballot.b32 %0, p, 0xffffffff;}"
                 : "=r"(ma) : "r"((unsigned)pa));
    asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; vote.sync.ballot.b32 %0, p, 0xffffffff;}"
                 : "=r"(mb) : "r"((unsigned)pb));
    const int na = __popc(ma);
#if PMC_QUEUE_PRED
    // predicated stores: only the ~7 % undecided samples move data
    if (pa) {
      const int sa = qn + __popc(ma & lt);
      qv[sa] = a0;
      qw[sa] = a1;
    }
    if (pb) {
      const int sb = qn + na + __popc(mb & lt);
      qv[sb] = b0;
      qw[sb] = b1;
    }
#else
    const int sa = pa ? qn + __popc(ma & lt) : QCAP + lane;
    const int sb = pb ? qn + na + __popc(mb & lt) : QCAP + lane;
    qv[sa] = a0;
    qw[sa] = a1;
    qv[sb] = b0;
    qw[sb] = b1;
#endif
    qn += na + __popc(mb);
  };
  auto push = [&](bool pend, const float4& st0, const float4& st1) {
    const unsigned pm = __ballot_sync(0xffffffffu, pend);
    const int slot = pend ? qn + __popc(pm & ((1u << lane) - 1u)) : QCAP + lane;
    qv[slot] = st0;
    qw[slot] = st1;
    qn += __popc(pm);
  };
  auto phase2 = [&](int slot, bool act) {
    if (act) {
      const float4 va = qv[slot], vb = qw[slot];
      const uint32_t s = __float_as_uint(vb.z);
      uint32_t r4, r5, r6, r7;
      philox4x32_10(c1, iso, c2, 2u * s + 1u, K, r4, r5, r6, r7);
      float z[8];
      upk(box_muller2(r4, r5, ONE), z[4], z[5]);
      upk(box_muller2(r6, r7, ONE), z[6], z[7]);
      float mx = vb.x, mn = vb.y;
      // y_c = (lo_c + B_c) + sum_{d>=4} L'_cd z_d, pairs (4,5) and (6,7)
      f2_t Y45 = ffma2(Q45[0], pk(z[4], z[4]), pk(va.x + B[0], va.y + B[1]));
      f2_t Y67 = pk(va.z + B[2], va.w + B[3]);
#pragma unroll
      for (int d = 4; d < 7; ++d) Y67 = ffma2(Q67[d - 4], pk(z[d], z[d]), Y67);
      float y[4];
      upk(Y45, y[0], y[1]);
      upk(Y67, y[2], y[3]);
      y[1] = fmaf(L55, z[5], y[1]);
      y[3] = fmaf(L77, z[7], y[3]);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        mx = fmaxf(mx, y[c]);
        mn = fminf(mn, y[c]);
      }
#pragma unroll
      for (int t = 0; t < T; ++t) cnt[t] += (mx >= dl(t) && mn <= dl(t)) ? 1u : 0u;
    }
  };
  auto drain = [&]() {
    if (qn >= 32) {
      __syncwarp();
      qn -= 32;
      phase2(qn + lane, true);
      p2 += 32;
      __syncwarp();
    }
  };
  uint32_t base = 0;
  // R13c: lane l takes the samples s = 128 h + l + 32 t, t = 0..3, of its group g = 32 h + l;
  // the group's phase-1 words are the 12 words of three Philox blocks with counters
  // (cell lo, iso, cell hi, 2 (3 g + j)), j = 0, 1, 2, and sample t takes words 3t..3t+2
  // (3 words = 4 uniforms of 23 bits: 3 Philox blocks per 4 samples instead of 4)
  auto group = [&](auto FULL) {
    constexpr bool full = decltype(FULL)::value;
    const uint32_t g = (base >> 2) + lane;   // 32 (base / 128) + lane
    uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
    philox4x32_10(c1, iso, c2, 2u * (3u * g), K, a0, a1, a2, a3);
    philox4x32_10(c1, iso, c2, 2u * (3u * g + 1u), K, b0, b1, b2, b3);
    float4 x0, x1, y0, y1;
    {
      const uint32_t sa = base + lane, sb = sa + 32u;
      const bool pa = phase1w(sa, a0, a1, a2, full || sa < Nl, x0, x1);
      const bool pb = phase1w(sb, a3, b0, b1, full || sb < Nl, y0, y1);
      if (ILP >= 2) {
        push2(pa, x0, x1, pb, y0, y1);
        drain();
        drain();
      } else {
        push(pa, x0, x1);
        drain();
        push(pb, y0, y1);
        drain();
      }
    }
    if (!full && base + 64u >= Nl) return;
    uint32_t e0, e1, e2, e3;
    philox4x32_10(c1, iso, c2, 2u * (3u * g + 2u), K, e0, e1, e2, e3);
    {
      const uint32_t sc = base + 64u + lane, sd = sc + 32u;
      const bool pc = phase1w(sc, b2, b3, e0, full || sc < Nl, x0, x1);
      const bool pd = phase1w(sd, e1, e2, e3, full || sd < Nl, y0, y1);
      if (ILP >= 2) {
        push2(pc, x0, x1, pd, y0, y1);
        drain();
        drain();
      } else {
        push(pc, x0, x1);
        drain();
        push(pd, y0, y1);
        drain();
      }
    }
  };
  for (; base + 128u <= Nl; base += 128u) group(std::true_type{});
  if (base < Nl) group(std::false_type{});   // a partial group: samples s >= N neither count nor queue
  if (qn > 0) {
    __syncwarp();
    phase2(lane, lane < qn);
    p2 += qn;
  }
  const uint32_t mk = (live && mask) ? mask[q] : 0xffffffffu;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const uint32_t ct = warp_sum(cnt[t]);
    if (live && lane == 0 && t < D.n_out) out[t * out_stride + q] = ((mk >> t) & 1u) ? (float)((double)ct / (double)N) : 0.0f;
  }
  if (live && lane == 0) atomicAdd(&s_p2, p2);
  __syncthreads();
  if (threadIdx.x == 0 && s_p2) atomicAdd(n_phase2, (unsigned long long)s_p2);
}

__global__ void k_scatter(const int64_t* __restrict__ cells, const float* __restrict__ lcp, int64_t n,
                          int64_t ncell, float* __restrict__ field, int* __restrict__ derr) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int64_t cell = cells[q];
  if (cell < 0 || cell >= ncell) atomicOr(derr, DERR_OVERFLOW);   // skipped, reported by the next check
  else field[cell] = lcp[q];
}

// posterior of n cells (device list) into post (n x 44 doubles); groups by
// bucket unless the list already comes in long same-bucket runs.
lcp_status_t posterior_impl(Ctx& c, const int64_t* cells, int64_t n, double* post) {
  NvtxRange nvtx_("leaf posterior");
  cudaError_t e;
#define CK(x)                                        \
  do {                                               \
    e = (x);                                         \
    if (e != cudaSuccess) return cuda_err(c, e, #x); \
  } while (0)
  if (n <= 0) return LCP_OK;
  CK(c.cell_bucket.ensure(sizeof(int32_t) * 2 * n));
  CK(c.counters.ensure(sizeof(unsigned long long) * 16));
  if (!c.h_counters) CK(cudaMallocHost(&c.h_counters, sizeof(int64_t) * 16));
  int32_t* bkt = c.cell_bucket.as<int32_t>();
  unsigned gr = (unsigned)((n + 255) / 256);
  k_cell_bucket<<<gr, 256, 0, c.stream>>>(c.g, cells, n, bkt, c.derr.as<int>());
  ++c.n_launch;
  // reject out-of-range ids before any brick kernel indexes by them
  if (lcp_status_t st = check_device_errors(c); st != LCP_OK) return st;
  c.last_brick_runs = 0;
  static const bool force_cell = [] {
    const char* v = std::getenv("LCP_POSTERIOR");
    return v && std::strcmp(v, "cell") == 0;
  }();
  if (!force_cell && c.opts.precision != LCP_FP32) {
    cudaError_t be;
    if (brick_posterior(c, cells, n, post, be)) return LCP_OK;
    if (be != cudaSuccess) return cuda_err(c, be, "brick posterior");
    if (brick_posterior_big(c, cells, n, post, be)) return LCP_OK;
    if (be != cudaSuccess) return cuda_err(c, be, "big-k brick posterior");
  }
  unsigned long long* dcnt = c.counters.as<unsigned long long>();
  CK(cudaMemsetAsync(dcnt + 15, 0, sizeof(unsigned long long), c.stream));
  k_count_runs<<<gr, 256, 0, c.stream>>>(bkt, n, dcnt + 15);
  ++c.n_launch;
  CK(cudaMemcpyAsync(c.h_counters + 15, dcnt + 15, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  int64_t runs = c.h_counters[15] + 1;
  if (n / runs >= 64 || c.g.nbuckets == 1) {
    CK(launch_cell_posterior(c, cells, nullptr, bkt, n, post));
  } else {
    CK(c.perm.ensure(sizeof(int64_t) * n));
    CK(group_by_bucket(c, bkt, n, c.perm.as<int64_t>()));
    int32_t* bs = bkt + n;
    k_gather_bkt<<<gr, 256, 0, c.stream>>>(bkt, c.perm.as<int64_t>(), n, bs);
    ++c.n_launch;
    CK(launch_cell_posterior(c, cells, c.perm.as<int64_t>(), bs, n, post));
  }
#undef CK
  return LCP_OK;
}

template <int T>
static void launch_pmc(Ctx& c, unsigned grid, const int64_t* cells, const double* post, int64_t rec_stride,
                       int by_morton, int64_t n, double theta, const IsoOffsets& D, uint32_t N,
                       const PhiloxKeys& keys, uint32_t iso, const uint32_t* mask, int64_t stride, float* out) {
  k_pmc<T><<<grid, PMC_WARPS * 32, 0, c.stream>>>(c.g, cells, post, rec_stride, by_morton, n, theta, D, N, keys, iso,
                                                  mask, stride, out, c.pmc_counters.as<unsigned long long>());
}

// leaf pass for T isovalues (T = 1: lcp_pmc_cells; T > 1: NEXT-3).  out[t * stride + q].
lcp_status_t pmc_multi_impl(Ctx& c, const int64_t* cells, int64_t n, const double* thetas, int T,
                            const uint32_t* mask, int64_t N, uint64_t seed, uint32_t iso, float* out,
                            int64_t stride) {
  NvtxRange nvtx_("lcp_pmc (T isovalues = %d)", T);
  if (!c.fitted) return set_err(c, LCP_ESTATE, "pmc before fit");
  if (N < 1 || N > ((int64_t)1 << 31)) return set_err(c, LCP_EINVAL, "pmc: need 1 <= n_samples <= 2^31");
  if (n < 0) return set_err(c, LCP_EINVAL, "pmc: negative cell count");
  if (T < 1 || T > MAX_ISO) return set_err(c, LCP_EINVAL, "pmc: need 1 <= n_iso <= 16");
  for (int t = 0; t < T; ++t)
    if (!std::isfinite(thetas[t])) return set_err(c, LCP_EINVAL, "pmc: isovalue not finite");
  if (n == 0) return LCP_OK;
  cudaError_t e;
#define CK(x)                                        \
  do {                                               \
    e = (x);                                         \
    if (e != cudaSuccess) return cuda_err(c, e, #x); \
  } while (0)
  if (!c.ev_init) {
    for (int i = 0; i < 8; ++i) cudaEventCreate(&c.ev[i]);
    c.ev_init = true;
  }
  CK(c.pmc_counters.ensure(sizeof(unsigned long long) * 2));
  CK(cudaMemsetAsync(c.pmc_counters.p, 0, sizeof(unsigned long long) * 2, c.stream));
  float tp = 0, tc = 0, tm = 0;
  PhiloxKeys keys;
  for (int r = 0; r < 10; ++r) {
    keys.k[2 * r] = (uint32_t)seed + (uint32_t)r * 0x9E3779B9u;
    keys.k[2 * r + 1] = (uint32_t)(seed >> 32) + (uint32_t)r * 0xBB67AE85u;
  }
  IsoOffsets D;
  for (int t = 0; t < MAX_ISO; ++t) D.dl[t] = t < T ? (float)(thetas[t] - thetas[0]) : INFINITY;
  D.n_out = T;
  D.one_bits = 0x3f800000u;
  const int Tp = T <= 4 ? T : (T <= 6 ? 6 : (T <= 8 ? 8 : (T <= 12 ? 12 : 16)));
  // records of the refine-time brick pass cover the list? (e.g. every leaf of a refine)
  bool use_rec = false;
  if (c.fused && c.rec_ready) {
    CK(c.counters.ensure(sizeof(unsigned long long) * 16));
    unsigned long long* dcnt = c.counters.as<unsigned long long>();
    CK(cudaMemsetAsync(dcnt + 12, 0, sizeof(unsigned long long), c.stream));
    k_cells_covered<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(c.g, cells, n, c.brick_done.as<uint8_t>(),
                                                                      dcnt + 12);
    ++c.n_launch;
    CK(cudaMemcpyAsync(c.h_counters + 12, dcnt + 12, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    use_rec = c.h_counters[12] == 0;
  }
  const int64_t chunk = use_rec ? n : std::min(n, PMC_CHUNK);
  if (!use_rec) CK(c.post.ensure(sizeof(double) * 44 * chunk));
  for (int64_t s0 = 0; s0 < n; s0 += chunk) {
    int64_t nn = std::min(chunk, n - s0);
    const double* rec = use_rec ? c.crec.as<double>() : c.post.as<double>();
    cudaEventRecord(c.ev[0], c.stream);
    if (!use_rec) {
      lcp_status_t st = posterior_impl(c, cells + s0, nn, c.post.as<double>());
      if (st != LCP_OK) return st;
    }
    cudaEventRecord(c.ev[1], c.stream);
    if (!use_rec) {
      k_chol8<<<(unsigned)((nn + 127) / 128), 128, 0, c.stream>>>(c.post.as<double>(), nn);
      ++c.n_launch;
    }
    cudaEventRecord(c.ev[2], c.stream);
    const unsigned gr = (unsigned)((nn + PMC_WARPS - 1) / PMC_WARPS);
    const uint32_t* mk = mask ? mask + s0 : nullptr;
    const int64_t rs = use_rec ? (int64_t)(sizeof(CellRec) / sizeof(double)) : 44;
    switch (Tp) {
#define LP(TT)                                                                                                  \
  case TT:                                                                                                      \
    launch_pmc<TT>(c, gr, cells + s0, rec, rs, use_rec ? 1 : 0, nn, thetas[0], D, (uint32_t)N, keys, iso, mk,  \
                   stride, out + s0);                                                                           \
    break
      LP(1); LP(2); LP(3); LP(4); LP(6); LP(8); LP(12); LP(16);
#undef LP
    }
    ++c.n_launch;
    cudaEventRecord(c.ev[3], c.stream);
    CK(cudaGetLastError());
    CK(cudaEventSynchronize(c.ev[3]));
    float a = 0, b = 0, d = 0;
    cudaEventElapsedTime(&a, c.ev[0], c.ev[1]);
    cudaEventElapsedTime(&b, c.ev[1], c.ev[2]);
    cudaEventElapsedTime(&d, c.ev[2], c.ev[3]);
    tp += a; tc += b; tm += d;
  }
  c.last_pmc_records = use_rec;
  c.t.posterior_ms = tp;
  c.t.chol_ms = tc;
  c.t.mc_ms = tm;
  c.last_pmc_cells = n;
  c.last_pmc_samples = n * N;
  CK(cudaMemcpy(&c.last_pmc_phase2, c.pmc_counters.p, sizeof(int64_t), cudaMemcpyDeviceToHost));
#undef CK
  return check_device_errors(c);
}

lcp_status_t pmc_impl(Ctx& c, const int64_t* cells, int64_t n, double theta, int64_t N, uint64_t seed,
                      uint32_t iso, float* out) {
  return pmc_multi_impl(c, cells, n, &theta, 1, nullptr, N, seed, iso, out, n);
}

cudaError_t launch_scatter(Ctx& c, const int64_t* cells, const float* lcp, int64_t n, float* field) {
  int64_t ncell = (int64_t)c.g.cells[0] * c.g.cells[1] * c.g.cells[2];
  cudaError_t e = cudaMemsetAsync(field, 0, sizeof(float) * ncell, c.stream);
  if (e != cudaSuccess) return e;
  if (n > 0) {
    k_scatter<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(cells, lcp, n, ncell, field, c.derr.as<int>());
    ++c.n_launch;
  }
  return cudaGetLastError();
}

}  // namespace lcp
