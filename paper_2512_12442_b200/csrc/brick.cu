// brick.cu -- leaf posterior on 4x4x4-cell bricks with FP64 tensor cores.
//
// Eq. 1 on the bucket's local GP, evaluated once per VERTEX of
// an aligned 4^3-cell brick instead of once per cell corner (the 8 corners of
// the 64 cells of a brick are only 125 distinct vertices):
//   phase 1  K[j][v] = k(x_j, v)            (k x 125, FP64, shared memory)
//            mu_v    = m0 + sum_j K[j][v] alpha_j
//   phase 2  V = L^-1 K                     (DMMA.8x8x4 FP64 tensor cores; L^-1 packed
//                                            lower triangle staged in shared memory)
//   phase 3  per leaf cell C of the brick:  Sigma_C = K_CC - V_C^T V_C  (DMMA, 8x8)
// The leaf list of lcp_octree_refine is in Morton order, so the leaves of one
// brick are contiguous; a CTA takes runs of one brick and keeps the bucket block
// staged while consecutive runs stay in the same bucket.  Identical arithmetic
// to k_cell_posterior up to FP64 rounding order.
#include <algorithm>
#include <cstdlib>

#include "chol8.cuh"
#include "expfast.cuh"

#include "ctx.h"

namespace lcp {

constexpr int BK = 4;                      // cells per brick side
constexpr int NVB = (BK + 1) * (BK + 1) * (BK + 1);   // 125 vertices
constexpr int NVP = 128;                    // padded vertex columns
// K/V row stride in doubles: 132 = 4 mod 16, so the four rows of a B fragment
// fall on disjoint bank octets within each half-warp phase (conflict-free).
constexpr int VSTR = 132;
constexpr int BRICK_THREADS = 512;          // 16 warps = 4 row sets x 4 column blocks of 32
#ifndef BRICK_CHUNK_N   // 8: a bucket block is staged once per 8 bricks (c5 brick pass 389.3 -> 387.2 ms; 16: 388.5)
#define BRICK_CHUNK_N 8
#endif
constexpr int BRICK_CHUNK = BRICK_CHUNK_N;  // runs grabbed per atomic
// k_brick's CTA: BT threads = 4 column blocks x NRS row sets of warps; mu / variance dots
// split over DOTP threads per vertex column
#ifndef BRICK_NT
#define BRICK_NT 512
#endif
constexpr int BT = BRICK_NT;
constexpr int NRS = BT / 128;               // row sets (4 or 8)
constexpr int TPW = 16 / NRS;               // row tiles per warp (4 or 2)
constexpr int DOTP = BT / NVP;              // threads per column in the mu / variance dots
constexpr int P1_UNROLL = BT >= 1024 ? 2 : 4;
// Timing-decomposition knobs (tools/brick_variants.py only; the records they produce are
// wrong): BRICK_DIAG_K = 1 replaces the kernel evaluation by one FMA on r^2,
// BRICK_DIAG_SOLVE = 0 / BRICK_DIAG_SIGMA = 0 skip the DMMA loops of phases 2 / 3.
#ifndef BRICK_DIAG_K
#define BRICK_DIAG_K 0
#endif
#ifndef BRICK_DIAG_SOLVE
#define BRICK_DIAG_SOLVE 1
#endif
#ifndef BRICK_DIAG_SIGMA
#define BRICK_DIAG_SIGMA 1
#endif
#ifndef BRICK_DIAG_MU       // 0: skip the mu dot
#define BRICK_DIAG_MU 1
#endif
#ifndef BRICK_DIAG_MARG     // 0: skip the vertex marginals
#define BRICK_DIAG_MARG 1
#endif
#ifndef BRICK_DIAG_REC      // 0: skip phase 3 (the per-cell records)
#define BRICK_DIAG_REC 1
#endif

// kernel value from r^2 (Matern-5/2 per BASELINE c4/c5) with exp_neg_fast
__device__ __forceinline__ double kern_from_r2_fast(const KernParams& p, double r2) {
  if (p.kind == LCP_K_SE) return p.var * exp_neg_fast(0.5 * r2);
  const double r = sqrt_fast(r2);
  const double s5 = SQRT5 * r;
  return p.var * (1.0 + s5 + (5.0 / 3.0) * r2) * exp_neg_fast(s5);
}
struct BrickArgs {
  KernParams kp;
  Geom g;
  int k, kp8;                 // k and k rounded up to a multiple of 8
  int64_t bstride;
  const double* bdata;
  double kcc[64];             // full 8x8 prior corner covariance
  double var_err;
};

__device__ __forceinline__ void dmma(double a, double b, double& d0, double& d1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ int64_t brick_key(const Geom& g, int64_t cell) {
  int i, j, k;
  cell_ijk(g, cell, i, j, k);
  return morton3(i / BK, j / BK, k / BK);
}

__global__ void k_brick_flags(Geom g, const int64_t* __restrict__ cells, int64_t n, int64_t* __restrict__ flag) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  flag[q] = (q == 0 || brick_key(g, cells[q]) != brick_key(g, cells[q - 1])) ? 1 : 0;
}

__global__ void k_brick_starts(const int64_t* __restrict__ flag, const int64_t* __restrict__ runidx, int64_t n,
                               int64_t* __restrict__ start) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n && flag[q]) start[runidx[q]] = q;
}

// Work unit of k_brick: a run of leaf cells of one brick (FUSED = false: the leaf
// pass of an arbitrary Morton-ordered list, output post[q]) or a whole brick given
// by its level-(Lfull-2) octree node key (FUSED = true: the refine-time brick pass,
// output post[64 u + local cell] for every in-grid cell of the brick, plus the
// vertex marginals of the brick's own-bucket vertices into the vertex cache).
struct BrickOut {
  double* post;               // 44 doubles per output slot
  double2* vcache;            // FUSED: (mu, 1 / (sigma sqrt 2)) per grid vertex
  uint32_t* vmask;            // FUSED: vertex "requested / cached" bits
  const uint64_t* bricks;     // FUSED: node keys (i | j << 21 | k << 42) at level Lfull - 2
  uint8_t* bdone;             // FUSED: per brick (Morton index of the node): pass done
  uint8_t* ucomp;             // FUSED: per unit of this launch: computed here (else skipped)
  double var_floor;
  int* derr;
};

template <bool FUSED>
__global__ void __launch_bounds__(BT, 1)
    k_brick(BrickArgs a, const int64_t* __restrict__ cells, const int64_t* __restrict__ run_start, int64_t nruns,
            unsigned long long* __restrict__ work, BrickOut o) {
  extern __shared__ double smem[];
  const int k = a.k, KP = a.kp8;
  const int64_t LA = la_size(k);
  const int64_t head = (LA + 4 * (int64_t)k + 1) & ~1ll;
  double* sLA = smem;
  double* sAlpha = smem + LA;
  double* sX = sAlpha + k;
  double* KV = smem + head;                     // KP x VSTR
  double* sMu = KV + (int64_t)KP * VSTR;        // NVP
  const int k16 = (k + 15) & ~15;               // sT rows: k rounded up to 16 (zero padding)
  double* sT = sMu + NVP;                       // k16 x 16: separable squared offsets (phase 1)
  double* sExp = sT + 16 * (int64_t)k16;        // 64: 2^(j/64) for exp_neg_tab
  __shared__ int64_t s_r0;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const Geom& g = a.g;
  if (tid < 64) sExp[tid] = c_exp2_64[tid];   // read after the loop's first barrier
  for (int64_t e = tid; e < (int64_t)KP * VSTR; e += BT) KV[e] = 0.0;   // padding rows / columns
  int staged = -1;
  // FUSED: thread 0 walks the unit list one brick ahead -- it grabs chunks, skips empty
  // slots and bricks done by an earlier refine, claims the next brick (bdone) during the
  // current brick's phase 3 and publishes it in s_ur / s_uk[(it + 1) & 1], so that the
  // dependent global round trips overlap the tensor-core work instead of stalling the CTA
  __shared__ int64_t s_ur[2];
  __shared__ uint64_t s_uk[2];
  int64_t tr = -1, trend = -1;
  auto claim_next = [&](int slot) {
    for (;;) {
      if (++tr >= trend) {
        tr = (int64_t)atomicAdd(work, (unsigned long long)BRICK_CHUNK);
        trend = min(nruns, tr + BRICK_CHUNK);
        if (tr >= nruns) {
          s_ur[slot] = -1;
          return;
        }
      }
      const uint64_t key = o.bricks[tr];
      if (key == ~0ull) {   // a child slot outside the grid (early pass)
        o.ucomp[tr] = 0;
        continue;
      }
      int bi, bj, bk;
      node_unkey(key, bi, bj, bk);
      uint8_t* d = o.bdone + (rec_index(g, BK * bi, BK * bj, BK * bk) >> 6);
      const uint8_t done = *d;
      *d = 1;
      o.ucomp[tr] = done ? 0 : 1;
      if (done) continue;   // done by an earlier refine (another isovalue)
      s_ur[slot] = tr;
      s_uk[slot] = key;
      return;
    }
  };
  if (FUSED) {
    if (tid == 0) claim_next(0);
    __syncthreads();
  }
  for (int it = 0;; ++it) {
    int64_t r0, r1;
    if (FUSED) {
      r0 = s_ur[it & 1];   // published before the previous brick's last barrier
      if (r0 < 0) break;
      r1 = r0 + 1;
    } else {
      if (tid == 0) s_r0 = (int64_t)atomicAdd(work, (unsigned long long)BRICK_CHUNK);
      __syncthreads();
      r0 = s_r0;
      if (r0 >= nruns) break;
      r1 = min(nruns, r0 + BRICK_CHUNK);
    }
    for (int64_t r = r0; r < r1; ++r) {
      int i0, j0, k0;
      int64_t q0 = 0, q1 = 0;
      if (FUSED) {
        int bi, bj, bk;
        node_unkey(s_uk[it & 1], bi, bj, bk);
        i0 = BK * bi; j0 = BK * bj; k0 = BK * bk;
      } else {
        q0 = run_start[r];
        q1 = run_start[r + 1];
        int ci, cj, ck;
        cell_ijk(g, cells[q0], ci, cj, ck);
        i0 = ci & ~(BK - 1); j0 = cj & ~(BK - 1); k0 = ck & ~(BK - 1);
      }
      // all cells of a brick lie in one bucket (bucket side >= BK)
      const int b = bucket_id(g, vbucket_axis(g, 0, i0), vbucket_axis(g, 1, j0), vbucket_axis(g, 2, k0));
      if (b != staged) {
        const double2* src = reinterpret_cast<const double2*>(a.bdata + (int64_t)b * a.bstride);
        double2* dst = reinterpret_cast<double2*>(smem);
        for (int64_t t = tid; t < (a.bstride >> 1); t += BT) dst[t] = __ldg(src + t);
        staged = b;
      }
      __syncthreads();   // (kept when nothing was staged: measured 1.3 ms faster on c5 than without)
      // phase 1: K[j][v] for the brick's (clamped) vertex lattice; zero padding.
      // r^2 is separable over the lattice: T[j][5d + t] = ((x_jd - v_d(t)) / l_d)^2 for the
      // 5 lattice positions t per axis d, then r^2 = (T_x + T_y) + T_z per element.
      for (int e = tid; e < 15 * k16; e += BT) {
        const int j = e / 15, col = e - 15 * j, d = col / 5, t = col - 5 * d;
        const int c0 = d == 0 ? i0 : (d == 1 ? j0 : k0);
        const double diff = j < k ? (sX[d * k + j] - vpos(g, d, min(c0 + t, g.cells[d]))) * a.kp.inv_ls[d] : 0.0;
        sT[16 * j + col] = diff * diff;
      }
      __syncthreads();
      {
        // branch-free kernel values (the kernel kind hoisted out of the loop, exp_neg_tab_bf
        // without the underflow branch, sqrt of r^2 + 1e-300 without the zero select) so
        // that the unrolled evaluations interleave; rows j >= k and the padding columns
        // v >= 125 are never written here: zeroed at kernel start, and the V write-back
        // (L^-1 times zero columns, zero rows of L^-1) keeps them zero
        const int v = tid & (NVP - 1);
        const int va = v % (BK + 1), vb = (v / (BK + 1)) % (BK + 1), vc = v / ((BK + 1) * (BK + 1));
        const bool vok = v < NVB;
        const int ta = vok ? va : 0, tb = vok ? 5 + vb : 5, tc = vok ? 10 + vc : 10;
        const double var = a.kp.var;
        // P1_UNROLL rows per step evaluated unconditionally (rows past k clamped, not
        // stored): a straight-line block the scheduler can interleave
        auto p1 = [&](auto kval) {
          constexpr int RS = BT / NVP;   // row stride of a thread
          for (int jb = tid >> 7; jb < k; jb += RS * P1_UNROLL) {
            double val[P1_UNROLL];
#pragma unroll
            for (int u = 0; u < P1_UNROLL; ++u) {
              const double* tj = sT + 16 * (jb + RS * u);   // rows up to k16: padding zeros
              val[u] = kval((tj[ta] + tj[tb]) + tj[tc]);
            }
#pragma unroll
            for (int u = 0; u < P1_UNROLL; ++u)
              if (vok && jb + RS * u < k) KV[(int64_t)(jb + RS * u) * VSTR + v] = val[u];
          }
        };
#if BRICK_DIAG_K
        p1([&](double r2) { return fma(r2, -1e-3, var); });
#else
        if (a.kp.kind == LCP_K_SE) {
          p1([&](double r2) { return var * exp_neg_tab_bf(0.5 * r2, sExp); });
        } else {
          p1([&](double r2) {
            const double r = sqrt_pos(r2 + 1e-300);
            const double s5 = SQRT5 * r;
            return var * (1.0 + s5 + (5.0 / 3.0) * r2) * exp_neg_tab_bf(s5, sExp);
          });
        }
#endif
      }
      __syncthreads();
      {
        // mu_v = m0 + sum_j K[j][v] alpha_j: 4 threads per vertex column (rows j = part
        // mod 4, conflict-free), combined as ((s0 + s1) + (s2 + s3))
        const int v = tid / DOTP, part = tid % DOTP;
        double s = 0.0;
        for (int j = part; j < (BRICK_DIAG_MU ? k : 0); j += DOTP) s = fma(KV[(int64_t)j * VSTR + v], sAlpha[j], s);
#pragma unroll
        for (int o = 1; o < DOTP; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (part == 0) sMu[v] = a.kp.m0 + s;
      }
      // phase 2: V = L^-1 K with DMMA; warp = (row set rs, column block cb)
      const int rs = wid >> 2, cb = wid & 3;
      const int nrt = KP >> 3;
      double acc[TPW][4][2];
#pragma unroll
      for (int t = 0; t < TPW; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
      const int lr = lane >> 2, lc = lane & 3;
      // row tiles rt(t) zig-zag over the NRS row sets so that every warp gets the same
      // triangular work (NRS = 4: rs = 0: 0, 7, 8, 15; rs = 3: 3, 4, 11, 12)
      auto rtile = [&](int t) { return (t & 1) ? (NRS - 1 - rs) + NRS * t : rs + NRS * t; };
      int last_rt = -1;
#pragma unroll
      for (int t = 0; t < TPW; ++t)
        if (rtile(t) < nrt) last_rt = max(last_rt, rtile(t));
      const int jend = (last_rt < 0 || !BRICK_DIAG_SOLVE) ? 0 : min(KP, 8 * last_rt + 8);
      // row tile by row tile: one A pointer live at a time (the accumulators of all four
      // tiles stay in registers until the write-back), B fragments re-read per tile
      const uint32_t kv_s = (uint32_t)__cvta_generic_to_shared(KV) + 8u * (lc * VSTR + 32 * cb + lr);
      const uint32_t la_s = (uint32_t)__cvta_generic_to_shared(sLA) + 8u * lane;
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        const int rt = rtile(t);
        const int je = (rt < nrt && BRICK_DIAG_SOLVE) ? 8 * rt + 8 : 0;
        const uint32_t pa = la_s + 8u * (uint32_t)la_block(rt < nrt ? rt : 0, 0);
#pragma unroll 2
        for (int j = 0; j < je; j += 4) {
          const uint32_t kb = kv_s + 8u * VSTR * j;
          const double af = lds_f64(pa + 64u * j);
#pragma unroll
          for (int u = 0; u < 4; ++u) dmma(af, lds_f64(kb + 64u * u), acc[t][u][0], acc[t][u][1]);
        }
      }
      __syncthreads();   // every warp has read K
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        const int rt = rtile(t);
        if (rt >= nrt) continue;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          double2* d = reinterpret_cast<double2*>(KV + (int64_t)(8 * rt + lr) * VSTR + 32 * cb + 8 * u + 2 * lc);
          *d = make_double2(acc[t][u][0], acc[t][u][1]);
        }
      }
      __syncthreads();
      if (FUSED && tid == 0) claim_next((it + 1) & 1);
      if (FUSED && BRICK_DIAG_MARG) {
        // vertex marginals (R10) of the brick's vertices whose own bucket is b:
        // var = k(v,v) - ||V_{:,v}||^2 (4 threads per column as for mu), cached as
        // (mu, 1 / (sigma sqrt 2))
        const int v = tid / DOTP, part = tid % DOTP;
        double s2 = 0.0;
        if (v < NVB)
          for (int j = part; j < k; j += DOTP) {
            const double x = KV[(int64_t)j * VSTR + v];
            s2 = fma(x, x, s2);
          }
#pragma unroll
        for (int o = 1; o < DOTP; o <<= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        if (part == 0 && v < NVB) {
          const int va = v % (BK + 1), vb = (v / (BK + 1)) % (BK + 1), vc = v / ((BK + 1) * (BK + 1));
          const int vi = i0 + va, vj = j0 + vb, vk = k0 + vc;
          if (vi <= g.cells[0] && vj <= g.cells[1] && vk <= g.cells[2] &&
              bucket_id(g, vbucket_axis(g, 0, vi), vbucket_axis(g, 1, vj), vbucket_axis(g, 2, vk)) == b) {
            const int64_t vid = vertex_id(g, vi, vj, vk);
            const uint32_t bit = 1u << (vid & 31);
            if (!(atomicOr(&o.vmask[vid >> 5], bit) & bit)) {
              const double var = a.kp.var - s2;
              if (var < a.var_err) atomicOr(o.derr, DERR_NUMERIC);
              const double vf = var > o.var_floor ? var : o.var_floor;
              o.vcache[vid] = make_double2(sMu[v], 1.0 / (sqrt(vf) * SQRT2));
            }
          }
        }
      }
      // phase 3: Sigma_C = K_CC - V_C^T V_C per cell (warp per cell)
      const int64_t nq = !BRICK_DIAG_REC ? 0 : FUSED ? BK * BK * BK : q1 - q0;
      for (int64_t qq = wid; qq < nq; qq += BT / 32) {
        int xi, xj, xk;
        int64_t slot;
        if (FUSED) {
          xi = i0 + (int)(qq & 3); xj = j0 + (int)((qq >> 2) & 3); xk = k0 + (int)(qq >> 4);
          if (xi >= g.cells[0] || xj >= g.cells[1] || xk >= g.cells[2]) continue;
          slot = 64 * r + qq;   // unit r of this launch
        } else {
          cell_ijk(g, cells[q0 + qq], xi, xj, xk);
          slot = q0 + qq;
        }
        const int cr = lr;   // corner of this lane's A row / B column
        const int lv = (xi - i0 + (cr & 1)) + (BK + 1) * ((xj - j0 + ((cr >> 1) & 1)) + (BK + 1) * (xk - k0 + (cr >> 2)));
        double d0 = 0.0, d1 = 0.0;
        {
          // two independent accumulator chains (even / odd k-steps), summed at the end
          // (c5 brick pass 401.8 -> 394.9 ms; four chains: 407 ms)
          double e0 = 0.0, e1 = 0.0;
          const uint32_t vb = (uint32_t)__cvta_generic_to_shared(KV) + 8u * (lc * VSTR + lv);
          const int kend = BRICK_DIAG_SIGMA ? KP : 0;
          int s = 0;
          for (; s + 8 <= kend; s += 8) {
            const double v0 = lds_f64(vb + 8u * VSTR * s), v1 = lds_f64(vb + 8u * VSTR * (s + 4));
            dmma(v0, v0, d0, d1);
            dmma(v1, v1, e0, e1);
          }
          if (s < kend) {
            const double v0 = lds_f64(vb + 8u * VSTR * s);
            dmma(v0, v0, d0, d1);
          }
          d0 += e0;
          d1 += e1;
        }
        double* rec = o.post + 44 * slot;
        // lane holds D[cr][2 lc], D[cr][2 lc + 1]
        const int c0 = 2 * lc, c1 = 2 * lc + 1;
        if (c0 <= cr) {
          double s0 = a.kcc[cr * 8 + c0] - d0;
          rec[8 + cr * (cr + 1) / 2 + c0] = s0;
          if (c0 == cr && s0 < a.var_err) atomicOr(o.derr, DERR_NUMERIC);
        }
        if (c1 <= cr) {
          double s1 = a.kcc[cr * 8 + c1] - d1;
          rec[8 + cr * (cr + 1) / 2 + c1] = s1;
          if (c1 == cr && s1 < a.var_err) atomicOr(o.derr, DERR_NUMERIC);
        }
        if (lc == 0) rec[cr] = sMu[lv];
      }
      __syncthreads();
    }
  }
}

static BrickArgs brick_args(const Ctx& c) {
  BrickArgs a;
  a.kp = c.kp;
  a.g = c.g;
  a.k = c.k;
  a.kp8 = (c.k + 7) & ~7;
  a.bstride = c.bstride;
  a.bdata = c.bdata.as<double>();
  for (int p = 0; p < 8; ++p)
    for (int q = 0; q < 8; ++q) a.kcc[p * 8 + q] = c.kcc[p >= q ? p * (p + 1) / 2 + q : q * (q + 1) / 2 + p];
  a.var_err = -1e-8 * c.kp.var;
  return a;
}

static size_t brick_smem(int k) {
  const int kp8 = (k + 7) & ~7;
  const int64_t head = (la_size(k) + 4 * (int64_t)k + 1) & ~1ll;
  return sizeof(double) * (head + (int64_t)kp8 * VSTR + NVP + 16 * (int64_t)((k + 15) & ~15) + 64);
}

bool fused_brick_supported(const Ctx& c) {
  return c.k <= 128 && c.g.bs >= BK && brick_smem(c.k) + 64 <= 227 * 1024 && c.opts.precision != LCP_FP32 &&
         c.g.lfull >= 2;
}

// Enable the refine-time brick pass for this fit when the kernel supports the model;
// LCP_FUSED=0 in the environment disables it (A/B measurements).  The record table
// (208 B per cell) covers the rank's slab (Geom rec_*): the whole virtual cube on one
// rank, allocated here; under a z-slab decomposition it is allocated by records_setup
// once the first refine has placed the slab.
lcp_status_t fused_setup(Ctx& c) {
  c.fused = false;
  c.rec_ready = false;
  c.g.rec_ls = 0;
  c.g.rec_z0 = 0;
  c.g.rec_z1 = 1;
  static const bool env_off = [] {
    const char* v = std::getenv("LCP_FUSED");
    return v && v[0] == '0';
  }();
  if (env_off || c.opts.brick_pass < 0 || !fused_brick_supported(c)) return LCP_OK;
  c.fused = true;
  if (c.opts.slab_count > 1) return LCP_OK;   // records_setup at the slab plan
  return records_setup(c);
}

// Allocate (grow-only) and clear the MC record table and the per-brick done flags for
// the record range of Geom rec_*, when they fit in free HBM with 4 GB to spare;
// otherwise the brick pass is switched off for this fit (leaves take the per-leaf path).
lcp_status_t records_setup(Ctx& c) {
  c.rec_ready = false;
  if (!c.fused) return LCP_OK;
  const int64_t ncodes = rec_count(c.g);
  const int64_t nbr = ncodes >> 6;
  const size_t need = sizeof(CellRec) * (size_t)ncodes;
  if (c.crec.cap < need) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess || need + ((size_t)4 << 30) > fr + c.crec.cap) {
      cudaGetLastError();
      c.fused = false;
      return LCP_OK;
    }
    c.crec.release();
  }
  cudaError_t e;
  if ((e = c.crec.ensure(need)) != cudaSuccess) {
    cudaGetLastError();
    c.fused = false;
    return LCP_OK;   // not enough memory after all: the per-leaf path stays
  }
  if ((e = c.brick_done.ensure(std::max<int64_t>(nbr, 1))) != cudaSuccess) return cuda_err(c, e, "brick_done");
  if ((e = c.brick_unit.ensure(BRICK_PASS_CHUNK)) != cudaSuccess) return cuda_err(c, e, "brick_unit");
  if ((e = cudaMemsetAsync(c.brick_done.p, 0, std::max<int64_t>(nbr, 1), c.stream)) != cudaSuccess)
    return cuda_err(c, e, "brick_done");
  c.rec_ready = true;
  return LCP_OK;
}

// FUSED brick pass over nb frontier nodes of level Lfull - 2 (node keys), writing
// the 8-corner posteriors of their cells into post (44 doubles per slot, slot =
// 64 u + local cell for unit u) and their own-bucket vertex marginals into the
// vertex cache.  Bricks already done (bdone) are skipped (their slots untouched).
cudaError_t launch_brick_pass(Ctx& c, const uint64_t* bricks, int64_t nb, double* post) {
  if (nb <= 0) return cudaSuccess;
  cudaError_t err;
  if ((err = c.counters.ensure(sizeof(unsigned long long) * 16)) != cudaSuccess) return err;
  unsigned long long* dcnt = c.counters.as<unsigned long long>();
  if ((err = cudaMemsetAsync(dcnt + 13, 0, sizeof(unsigned long long), c.stream)) != cudaSuccess) return err;
  const size_t smem = brick_smem(c.k);
  if ((err = cudaFuncSetAttribute(k_brick<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return err;
  BrickOut o;
  o.post = post;
  o.vcache = c.vcache.as<double2>();
  o.vmask = c.vstate.as<uint32_t>();
  o.bricks = bricks;
  o.bdone = c.brick_done.as<uint8_t>();
  o.ucomp = c.brick_unit.as<uint8_t>();
  o.var_floor = 1e-12 * c.kp.var;
  o.derr = c.derr.as<int>();
  unsigned grid = (unsigned)std::min<int64_t>((nb + BRICK_CHUNK - 1) / BRICK_CHUNK, (int64_t)c.sm_count);
  k_brick<true><<<grid, BT, smem, c.stream>>>(brick_args(c), nullptr, nullptr, nb, dcnt + 13, o);
  ++c.n_launch;
  return cudaGetLastError();
}

// The 8^gen descendant bricks (level Lfull-2 node keys) of level-(Lfull-2-gen) frontier
// nodes, node by node; slots whose brick holds no grid cell get the key ~0 (skipped).
__global__ void k_child_bricks(Geom g, const uint64_t* __restrict__ F, int64_t nF, int gen,
                               uint64_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (nF << (3 * gen))) return;
  int i, j, k;
  node_unkey(F[t >> (3 * gen)], i, j, k);
  const int c = (int)(t & ((1 << (3 * gen)) - 1)), msk = (1 << gen) - 1;
  const int bi = (i << gen) + (c & msk), bj = (j << gen) + ((c >> gen) & msk), bk = (k << gen) + (c >> (2 * gen));
  const bool in = BK * bi < g.cells[0] && BK * bj < g.cells[1] && BK * bk < g.cells[2];
  out[t] = in ? node_key(bi, bj, bk) : ~0ull;
}

cudaError_t launch_child_bricks(Ctx& c, const uint64_t* F, int64_t nF, int gen, uint64_t* out) {
  if (nF <= 0) return cudaSuccess;
  const int64_t n = nF << (3 * gen);
  k_child_bricks<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(c.g, F, nF, gen, out);
  ++c.n_launch;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- big k
// k_brick_big: the brick posterior for 128 < k <= BIG_KMAX (e.g. the exact-GP dense
// baseline, k = m = 500), where neither K (k x 128) nor L^-1 fits in shared memory.
// Per brick the 125 vertex columns go in 4 chunks of 32: K chunk in smem (row stride
// 36 = 4 mod 16), V chunk = L^-1 K chunk by DMMA with the A fragments streamed from
// global memory (L2-resident, each feeding 4 column tiles), V stored column-major in a
// per-CTA global scratch (L2-resident); then Sigma_C = K_CC - V_C^T V_C per leaf cell
// of the run by DMMA on the scratch.  Leaves come through a permutation (grouped by
// brick); results go to post[perm[q]].
constexpr int BIG_KMAX = 640;
constexpr int BIG_CH = 32;                   // columns per chunk
constexpr int BIG_CST = 36;                  // K chunk row stride (doubles)

__global__ void __launch_bounds__(BRICK_THREADS, 1)
    k_brick_big(BrickArgs a, const int64_t* __restrict__ cells, const int64_t* __restrict__ perm,
                const int64_t* __restrict__ run_start, int64_t nruns, unsigned long long* __restrict__ work,
                double* __restrict__ vscratch, double* __restrict__ post, int* __restrict__ derr) {
  extern __shared__ double smem[];
  const int k = a.k, KP = a.kp8, NRT = KP >> 3;
  double* sAlpha = smem;                       // k
  double* sX = sAlpha + k;                     // 3k
  double* KC = smem + ((4 * (int64_t)k + 1) & ~1ll);   // KP x BIG_CST
  double* sMu = KC + (int64_t)KP * BIG_CST;    // NVP
  double* Vg = vscratch + (int64_t)blockIdx.x * NVP * KP;   // column-major: V[col][row]
  __shared__ int64_t s_r0;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const Geom& g = a.g;
  int staged = -1;
  const int nt = (NRT + 15) / 16;              // row tiles per warp (<= 5 for KP <= 640)
  for (;;) {
    if (tid == 0) s_r0 = (int64_t)atomicAdd(work, 1ull);
    __syncthreads();
    const int64_t r = s_r0;
    if (r >= nruns) break;
    const int64_t q0 = run_start[r], q1 = run_start[r + 1];
    int ci, cj, ck;
    cell_ijk(g, cells[perm[q0]], ci, cj, ck);
    const int i0 = ci & ~(BK - 1), j0 = cj & ~(BK - 1), k0 = ck & ~(BK - 1);
    const int b = bucket_id(g, vbucket_axis(g, 0, i0), vbucket_axis(g, 1, j0), vbucket_axis(g, 2, k0));
    const double* blk = a.bdata + (int64_t)b * a.bstride;
    if (b != staged) {
      for (int t = tid; t < 4 * k; t += BRICK_THREADS) smem[t] = __ldg(blk + la_size(k) + t);
      staged = b;
    }
    __syncthreads();
    for (int cc = 0; cc < NVP / BIG_CH; ++cc) {
      // K chunk: columns v = 32 cc + cl of the brick's (clamped) vertex lattice
      {
        const int cl = tid & (BIG_CH - 1), v = BIG_CH * cc + cl;
        const bool vok = v < NVB;
        const int va = v % (BK + 1), vb = (v / (BK + 1)) % (BK + 1), vc = v / ((BK + 1) * (BK + 1));
        const int vi = min(i0 + (vok ? va : 0), g.cells[0]), vj = min(j0 + (vok ? vb : 0), g.cells[1]),
                  vk = min(k0 + (vok ? vc : 0), g.cells[2]);
        const double px = vpos(g, 0, vi), py = vpos(g, 1, vj), pz = vpos(g, 2, vk);
        for (int j = tid / BIG_CH; j < KP; j += BRICK_THREADS / BIG_CH) {
          const int jj = min(j, k - 1);
          const double r2 = kern_r2(a.kp, sX[jj] - px, sX[k + jj] - py, sX[2 * k + jj] - pz);
          const double val = kern_from_r2_fast(a.kp, r2);
          KC[(int64_t)j * BIG_CST + cl] = (j < k && vok) ? val : 0.0;
        }
      }
      __syncthreads();
      {
        // mu of the chunk's columns: 16 threads per column
        const int cl = tid >> 4, part = tid & 15;
        double sacc = 0.0;
        for (int j = part; j < k; j += 16) sacc = fma(KC[(int64_t)j * BIG_CST + cl], sAlpha[j], sacc);
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
        if (part == 0) sMu[BIG_CH * cc + cl] = a.kp.m0 + sacc;
      }
      // V chunk = L^-1 K chunk: warp w owns row tiles w + 16 t (zig-zag), all 4 column tiles
      double acc[5][4][2];
#pragma unroll
      for (int t = 0; t < 5; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
      auto rtile = [&](int t) { return (t & 1) ? (15 - wid) + 16 * t : wid + 16 * t; };
      int last = -1;
#pragma unroll
      for (int t = 0; t < 5; ++t)
        if (t < nt && rtile(t) < NRT) last = max(last, rtile(t));
      const int jend = last < 0 ? 0 : min(KP, 8 * last + 8);
      const double* LA = blk;
      for (int j = 0; j < jend; j += 4) {
        double bf[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) bf[u] = KC[(int64_t)(j + lc) * BIG_CST + 8 * u + lr];
#pragma unroll
        for (int t = 0; t < 5; ++t) {
          const int rt = rtile(t);
          if (t >= nt || rt >= NRT || 8 * rt + 7 < j) continue;   // warp-uniform
          const double af = __ldg(LA + la_block(rt, j >> 2) + lane);
#pragma unroll
          for (int u = 0; u < 4; ++u) dmma(af, bf[u], acc[t][u][0], acc[t][u][1]);
        }
      }
#pragma unroll
      for (int t = 0; t < 5; ++t) {
        const int rt = rtile(t);
        if (t >= nt || rt >= NRT) continue;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int col = BIG_CH * cc + 8 * u + 2 * lc, row = 8 * rt + lr;
          Vg[(int64_t)col * KP + row] = acc[t][u][0];
          Vg[(int64_t)(col + 1) * KP + row] = acc[t][u][1];
        }
      }
      __syncthreads();   // KC is rewritten by the next chunk; V chunk visible to the block
    }
    // Sigma_C = K_CC - V_C^T V_C per leaf of the run (warp per cell)
    for (int64_t qq = q0 + wid; qq < q1; qq += BRICK_THREADS / 32) {
      const int64_t slot = perm[qq];
      int xi, xj, xk;
      cell_ijk(g, cells[slot], xi, xj, xk);
      const int cr = lr;
      const int lv = (xi - i0 + (cr & 1)) + (BK + 1) * ((xj - j0 + ((cr >> 1) & 1)) + (BK + 1) * (xk - k0 + (cr >> 2)));
      const double* vcol = Vg + (int64_t)lv * KP;
      double d0 = 0.0, d1 = 0.0;
      for (int sidx = 0; sidx < KP; sidx += 4) {
        const double v = vcol[sidx + lc];
        dmma(v, v, d0, d1);
      }
      double* rec = post + 44 * slot;
      const int c0 = 2 * lc, c1 = 2 * lc + 1;
      if (c0 <= cr) {
        const double s0 = a.kcc[cr * 8 + c0] - d0;
        rec[8 + cr * (cr + 1) / 2 + c0] = s0;
        if (c0 == cr && s0 < a.var_err) atomicOr(derr, DERR_NUMERIC);
      }
      if (c1 <= cr) {
        const double s1 = a.kcc[cr * 8 + c1] - d1;
        rec[8 + cr * (cr + 1) / 2 + c1] = s1;
        if (c1 == cr && s1 < a.var_err) atomicOr(derr, DERR_NUMERIC);
      }
      if (lc == 0) rec[cr] = sMu[lv];
    }
    __syncthreads();
  }
}

__global__ void k_brick_keys(Geom g, const int64_t* __restrict__ cells, int64_t n, int32_t* __restrict__ key) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) key[q] = (int32_t)brick_key(g, cells[q]);
}
__global__ void k_brick_flags_perm(const int32_t* __restrict__ key, const int64_t* __restrict__ perm, int64_t n,
                                   int64_t* __restrict__ flag) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  flag[q] = (q == 0 || key[perm[q]] != key[perm[q - 1]]) ? 1 : 0;
}

// big-k brick posterior of an arbitrary list: group the cells by brick, then
// k_brick_big over the runs.  Returns false (no error) when k is out of range or
// the list has fewer than 8 cells per brick on average.
bool brick_posterior_big(Ctx& c, const int64_t* cells, int64_t n, double* post, cudaError_t& err) {
  err = cudaSuccess;
  if (c.k <= 128 || c.k > BIG_KMAX || c.g.bs < BK || c.g.lfull < 2 || 3 * (c.g.lfull - 2) > 30) return false;
  const int k = c.k, kp8 = (k + 7) & ~7;
  const int64_t nbr = (int64_t)1 << (3 * (c.g.lfull - 2));
  // own key buffer: the caller's per-cell bucket ids (c.cell_bucket) must survive a
  // decline (too few cells per brick) for the per-cell fallback
  if ((err = c.brick_key.ensure(sizeof(int32_t) * n)) != cudaSuccess) return false;
  if ((err = c.perm.ensure(sizeof(int64_t) * n)) != cudaSuccess) return false;
  if ((err = c.brick_flag.ensure(sizeof(int64_t) * n)) != cudaSuccess) return false;
  if ((err = c.brick_idx.ensure(sizeof(int64_t) * n)) != cudaSuccess) return false;
  if ((err = c.gcount.ensure(sizeof(int64_t) * (nbr + 1))) != cudaSuccess) return false;
  if ((err = c.goff.ensure(sizeof(int64_t) * (nbr + 1))) != cudaSuccess) return false;
  if ((err = c.counters.ensure(sizeof(unsigned long long) * 16)) != cudaSuccess) return false;
  unsigned long long* dcnt = c.counters.as<unsigned long long>();
  int32_t* key = c.brick_key.as<int32_t>();
  int64_t* pm = c.perm.as<int64_t>();
  const unsigned gr = (unsigned)((n + 255) / 256);
  k_brick_keys<<<gr, 256, 0, c.stream>>>(c.g, cells, n, key);
  ++c.n_launch;
  if ((err = group_by_key(c, key, n, nbr, pm)) != cudaSuccess) return false;
  k_brick_flags_perm<<<gr, 256, 0, c.stream>>>(key, pm, n, c.brick_flag.as<int64_t>());
  ++c.n_launch;
  if ((err = exclusive_scan_i64(c, c.brick_flag.as<int64_t>(), c.brick_idx.as<int64_t>(), n,
                                (int64_t*)(dcnt + 14))) != cudaSuccess)
    return false;
  if ((err = cudaMemcpyAsync(c.h_counters + 14, dcnt + 14, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream)) !=
      cudaSuccess)
    return false;
  if ((err = cudaStreamSynchronize(c.stream)) != cudaSuccess) return false;
  const int64_t nruns = c.h_counters[14];
  if (n / std::max<int64_t>(nruns, 1) < 8) return false;
  if ((err = c.brick_start.ensure(sizeof(int64_t) * (nruns + 1))) != cudaSuccess) return false;
  int64_t* start = c.brick_start.as<int64_t>();
  k_brick_starts<<<gr, 256, 0, c.stream>>>(c.brick_flag.as<int64_t>(), c.brick_idx.as<int64_t>(), n, start);
  ++c.n_launch;
  if ((err = cudaMemcpyAsync(start + nruns, &n, sizeof(int64_t), cudaMemcpyHostToDevice, c.stream)) != cudaSuccess)
    return false;
  if ((err = cudaMemsetAsync(dcnt + 13, 0, sizeof(unsigned long long), c.stream)) != cudaSuccess) return false;
  const size_t smem = sizeof(double) * (((4 * (int64_t)k + 1) & ~1ll) + (int64_t)kp8 * BIG_CST + NVP);
  if ((err = cudaFuncSetAttribute(k_brick_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return false;
  const unsigned grid = (unsigned)std::min<int64_t>(nruns, (int64_t)c.sm_count);
  if ((err = c.vscratch.ensure(sizeof(double) * (size_t)grid * NVP * kp8)) != cudaSuccess) return false;
  k_brick_big<<<grid, BRICK_THREADS, smem, c.stream>>>(brick_args(c), cells, pm, start, nruns, dcnt + 13,
                                                       c.vscratch.as<double>(), post, c.derr.as<int>());
  ++c.n_launch;
  err = cudaGetLastError();
  c.last_brick_runs = nruns;
  return err == cudaSuccess;
}

// Returns true when the brick path handled the list (Morton-like order with
// enough leaves per brick and k small enough for shared memory).
bool brick_posterior(Ctx& c, const int64_t* cells, int64_t n, double* post, cudaError_t& err) {
  err = cudaSuccess;
  if (c.k > 128 || c.g.bs < BK) return false;
  const int k = c.k;
  size_t smem = brick_smem(k);
  if (smem + 64 > 227 * 1024) return false;
  if ((err = c.brick_flag.ensure(sizeof(int64_t) * n)) != cudaSuccess) return false;
  if ((err = c.brick_idx.ensure(sizeof(int64_t) * n)) != cudaSuccess) return false;
  if ((err = c.counters.ensure(sizeof(unsigned long long) * 16)) != cudaSuccess) return false;
  unsigned long long* dcnt = c.counters.as<unsigned long long>();
  unsigned gr = (unsigned)((n + 255) / 256);
  k_brick_flags<<<gr, 256, 0, c.stream>>>(c.g, cells, n, c.brick_flag.as<int64_t>());
  ++c.n_launch;
  if ((err = exclusive_scan_i64(c, c.brick_flag.as<int64_t>(), c.brick_idx.as<int64_t>(), n,
                                (int64_t*)(dcnt + 14))) != cudaSuccess)
    return false;
  if ((err = cudaMemcpyAsync(c.h_counters + 14, dcnt + 14, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream)) !=
      cudaSuccess)
    return false;
  if ((err = cudaStreamSynchronize(c.stream)) != cudaSuccess) return false;
  const int64_t nruns = c.h_counters[14];
  if (n / std::max<int64_t>(nruns, 1) < 8) return false;   // too few leaves per brick: per-cell kernel
  if ((err = c.brick_start.ensure(sizeof(int64_t) * (nruns + 1))) != cudaSuccess) return false;
  int64_t* start = c.brick_start.as<int64_t>();
  k_brick_starts<<<gr, 256, 0, c.stream>>>(c.brick_flag.as<int64_t>(), c.brick_idx.as<int64_t>(), n, start);
  ++c.n_launch;
  if ((err = cudaMemcpyAsync(start + nruns, &n, sizeof(int64_t), cudaMemcpyHostToDevice, c.stream)) != cudaSuccess)
    return false;
  if ((err = cudaMemsetAsync(dcnt + 13, 0, sizeof(unsigned long long), c.stream)) != cudaSuccess) return false;
  if ((err = cudaFuncSetAttribute(k_brick<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return false;
  BrickOut o{};
  o.post = post;
  o.derr = c.derr.as<int>();
  int blocks_per_sm = smem <= 110 * 1024 ? 2 : 1;
  unsigned grid = (unsigned)std::min<int64_t>((nruns + BRICK_CHUNK - 1) / BRICK_CHUNK, (int64_t)c.sm_count * blocks_per_sm);
  k_brick<false><<<grid, BT, smem, c.stream>>>(brick_args(c), cells, start, nruns, dcnt + 13, o);
  ++c.n_launch;
  err = cudaGetLastError();
  c.last_brick_runs = nruns;
  return err == cudaSuccess;
}

}  // namespace lcp
