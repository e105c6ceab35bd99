// extreme.cu -- NEXT-1: continuous refinement of a node's extreme
// probabilities ("any random variable Y continuously defined in the
// region", :183 quasi-Newton search with a closed-form gradient; reading R26).
//
// For nodes coarser than h_full (whose candidate lattice is strided) that need a
// bound, one warp per node climbs f(x) = (mu(x) - theta) / (sigma(x) sqrt 2) from
// the lattice argmax (for Q_lo) and descends from the lattice argmin (for Q_hi)
// over the node box with a deterministic projected limited-memory quasi-Newton
// iteration (L-BFGS two-loop direction on the free variables, projected Armijo
// backtracking; R26/R26b; the CPU oracle implements it independently).  Each evaluation of f and
// grad f at a point uses the bucket's local GP:
//   K columns [k_x, d k_x / dx_0, d/dx_1, d/dx_2] for both search points (8 columns),
//   mu and grad mu = the columns dotted with alpha,
//   V = L^-1 K and D = V^T V on the FP64 tensor cores (DMMA.8x8x4),
//   var = sigma_f^2 - D[v][v], grad var = -2 D[v][d_x].
// U is recomputed from the refined extremes (they can only move outward).
#include "ctx.h"

namespace lcp {

__device__ __forceinline__ void dmma_x(double a, double b, double& d0, double& d1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int EXT_MEM = 4;   // L-BFGS memory (pairs s, y) per search

struct ExtArgs {
  KernParams kp;
  Geom g;
  int k, ks, bucket_log2, iters;
  int64_t bstride, la;
  const double* bdata;
  double theta, alpha, var_floor;
};

// dk(x, xj)/dx (first argument), kernel value returned
__device__ __forceinline__ double kern_val_grad(const KernParams& p, const double* x, double xj, double yj, double zj,
                                                double* g) {
  double dx = x[0] - xj, dy = x[1] - yj, dz = x[2] - zj;
  double r2 = kern_r2(p, dx, dy, dz);
  double kv, c;
  if (p.kind == LCP_K_SE) {
    kv = p.var * exp(-0.5 * r2);
    c = -kv;
  } else {
    double r = sqrt(r2), s = SQRT5 * r, e = exp(-s);
    kv = p.var * (1.0 + s + (5.0 / 3.0) * r2) * e;
    c = -(5.0 / 3.0) * p.var * (1.0 + s) * e;
  }
  g[0] = c * dx * p.inv_ls[0] * p.inv_ls[0];
  g[1] = c * dy * p.inv_ls[1] * p.inv_ls[1];
  g[2] = c * dz * p.inv_ls[2] * p.inv_ls[2];
  return kv;
}

// f and grad f at the points x[p] (p < np <= 2) of bucket b; all lanes get the results.
__device__ void eval_f_grad(const ExtArgs& a, int b, const double (&x)[2][3], int np, double* sK, double* sV,
                            double (&f)[2], double (&gf)[2][3]) {
  const int k = a.k, ks = a.ks;
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  const double* blk = a.bdata + (int64_t)b * a.bstride;
  const double* LA = blk;
  const double* alpha = blk + a.la;
  const double* Xs = alpha + k;
  for (int j = lane; j < k; j += 32) {
    const double xj = Xs[j], yj = Xs[k + j], zj = Xs[2 * k + j];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      double g[3] = {0.0, 0.0, 0.0}, kv = 0.0;
      if (p < np) kv = kern_val_grad(a.kp, x[p], xj, yj, zj, g);
      sK[(4 * p + 0) * ks + j] = kv;
      sK[(4 * p + 1) * ks + j] = g[0];
      sK[(4 * p + 2) * ks + j] = g[1];
      sK[(4 * p + 3) * ks + j] = g[2];
    }
  }
  __syncwarp();
  // column dots with alpha: lane c = lane & 7 after the reduction
  double dotc;
  {
    int c = lane & 7, part = lane >> 3;
    double s = 0.0;
    for (int j = part; j < k; j += 4) s = fma(sK[c * ks + j], alpha[j], s);
    s += __shfl_xor_sync(0xffffffffu, s, 8);
    s += __shfl_xor_sync(0xffffffffu, s, 16);
    dotc = s;
  }
  // V = L^-1 K by row groups of 128, D = V^T V
  double o0 = 0.0, o1 = 0.0;
  const bool single = k <= 128;
  for (int row0 = 0; row0 < k; row0 += 128) {
    double acc[16][2];
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t][0] = acc[t][1] = 0.0;
    const int nrows = min(128, k - row0), nrt = (nrows + 7) >> 3, rt0 = row0 >> 3;
    for (int j = 0; j < row0 + 8 * nrt; j += 4) {
      const int jj = j + lc, js = j >> 2;
      const double bb = jj < k ? sK[lr * ks + jj] : 0.0;
      const int rt_lo = j < row0 ? 0 : ((j - row0) >> 3);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        if (t < rt_lo || t >= nrt) continue;
        dmma_x(LA[la_block(rt0 + t, js) + lane], bb, acc[t][0], acc[t][1]);
      }
    }
    double* dst = single ? sK : sV;
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int r = 8 * t + lr;
      if (r < nrows) *reinterpret_cast<double2*>(dst + 8 * r + 2 * lc) = make_double2(acc[t][0], acc[t][1]);
    }
    __syncwarp();
    for (int s = 0; s < nrows; s += 4) {
      const int r = s + lc;
      const double v = r < nrows ? dst[8 * r + lr] : 0.0;
      dmma_x(v, v, o0, o1);
    }
    __syncwarp();
  }
  // lane holds D[lr][2 lc + e]; point p needs D[4p][4p + q], q = 0..3 (row 4p, lanes 16p + 2p'..)
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const int r = 4 * p;
    // D[r][4p + q]: lane = 4 r + (4p + q) / 2, element (4p + q) & 1
    double dq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int col = 4 * p + q;
      const double e0 = __shfl_sync(0xffffffffu, o0, 4 * r + col / 2);
      const double e1 = __shfl_sync(0xffffffffu, o1, 4 * r + col / 2);
      dq[q] = (col & 1) ? e1 : e0;
    }
    double mu = a.kp.m0 + __shfl_sync(0xffffffffu, dotc, 4 * p);
    double gmu[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) gmu[d] = __shfl_sync(0xffffffffu, dotc, 4 * p + 1 + d);
    const double var = a.kp.var - dq[0];
    const double vf = var > a.var_floor ? var : a.var_floor, s = sqrt(vf);
    f[p] = (mu - a.theta) / (s * SQRT2);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double gs = var > a.var_floor ? (-2.0 * dq[1 + d]) / (2.0 * s) : 0.0;
      gf[p][d] = (gmu[d] * s - (mu - a.theta) * gs) / (vf * SQRT2);
    }
  }
}

__global__ void __launch_bounds__(256) k_node_extreme(ExtArgs a, int level, const uint64_t* __restrict__ front,
                                                      int64_t nF, const int8_t* __restrict__ ncase,
                                                      int8_t* __restrict__ nref, double* __restrict__ nU,
                                                      const double* __restrict__ ext_z,
                                                      const int64_t* __restrict__ ext_v) {
  extern __shared__ double smem[];
  const int64_t n = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int wid = threadIdx.x >> 5;
  if (n >= nF) return;
  const int cs = ncase[n];
  if (cs == 1) return;   // warp-uniform
  const Geom& g = a.g;
  const int per_warp = 8 * a.ks + (a.k > 128 ? 1024 : 0);
  double* sK = smem + (int64_t)wid * per_warp;
  double* sV = sK + 8 * a.ks;
  int ni, nj, nk;
  node_unkey(front[n], ni, nj, nk);
  const int h = g.lfull - level;
  int64_t base[3] = {(int64_t)ni << h, (int64_t)nj << h, (int64_t)nk << h};
  int64_t vmax[3];
  for (int d = 0; d < 3; ++d) {
    int64_t e = base[d] + ((int64_t)1 << h);
    vmax[d] = e < g.cells[d] ? e : g.cells[d];
  }
  // per side s (0: maximise f for Q_lo, 1: minimise f for Q_hi): bucket, box, start
  int bk[2];
  double blo[2][3], bhi[2][3], x[2][3], step[2], smax[2];
  for (int s = 0; s < 2; ++s) {
    int av[3];
    vertex_ijk(g, ext_v[2 * n + s], av[0], av[1], av[2]);
    int64_t lo_v[3], hi_v[3];
    if (level >= a.bucket_log2) {
      bk[s] = bucket_id(g, vbucket_axis(g, 0, base[0]), vbucket_axis(g, 1, base[1]), vbucket_axis(g, 2, base[2]));
      for (int d = 0; d < 3; ++d) { lo_v[d] = base[d]; hi_v[d] = vmax[d]; }
    } else {
      int bi[3] = {vbucket_axis(g, 0, av[0]), vbucket_axis(g, 1, av[1]), vbucket_axis(g, 2, av[2])};
      bk[s] = bucket_id(g, bi[0], bi[1], bi[2]);
      for (int d = 0; d < 3; ++d) {
        int64_t b0 = (int64_t)bi[d] * g.bs, b1 = b0 + g.bs;
        lo_v[d] = base[d] > b0 ? base[d] : b0;
        hi_v[d] = vmax[d] < b1 ? vmax[d] : b1;
      }
    }
    double mn = INFINITY, mx = 0.0;
    for (int d = 0; d < 3; ++d) {
      blo[s][d] = vpos(g, d, lo_v[d]);
      bhi[s][d] = vpos(g, d, hi_v[d]);
      x[s][d] = vpos(g, d, av[d]);
      double w = bhi[s][d] - blo[s][d];
      mn = fmin(mn, w);
      mx = fmax(mx, w);
    }
    step[s] = 0.25 * mn;   // the first step length (no curvature memory yet)
    smax[s] = mx;
  }
  const double sg[2] = {1.0, -1.0};
  double F[2], gr[2][3], f[2], gf[2][3];
  // starting values (both sides share a bucket when the node lies in one)
  if (bk[0] == bk[1]) {
    eval_f_grad(a, bk[0], x, 2, sK, sV, f, gf);
  } else {
    double xs[2][3] = {{x[1][0], x[1][1], x[1][2]}, {0, 0, 0}}, f1[2], gf1[2][3];
    eval_f_grad(a, bk[0], x, 1, sK, sV, f, gf);
    eval_f_grad(a, bk[1], xs, 1, sK, sV, f1, gf1);
    f[1] = f1[0];
    for (int d = 0; d < 3; ++d) gf[1][d] = gf1[0][d];
  }
  // R26b: projected limited-memory quasi-Newton ascent of F = sg f per side (the CPU
  // oracle implements the same iteration independently)
  double Sm[2][EXT_MEM][3], Ym[2][EXT_MEM][3], RHO[2][EXT_MEM], dir[2][3], t[2], dn[2];
  int nmem[2] = {0, 0};
  bool done[2], need_dir[2] = {true, true};
  for (int s = 0; s < 2; ++s) {
    F[s] = sg[s] * f[s];
    for (int d = 0; d < 3; ++d) gr[s][d] = sg[s] * gf[s][d];
    done[s] = false;
    t[s] = dn[s] = 0.0;
  }
  for (int it = 0; it < a.iters && !(done[0] && done[1]); ++it) {
    double xn[2][3];
    for (int s = 0; s < 2; ++s) {
      for (int d = 0; d < 3; ++d) xn[s][d] = x[s][d];
      while (!done[s]) {                 // find a trial point (no evaluation)
        if (need_dir[s]) {
          double gfr[3];
          for (int d = 0; d < 3; ++d)
            gfr[d] = ((x[s][d] <= blo[s][d] && gr[s][d] < 0.0) || (x[s][d] >= bhi[s][d] && gr[s][d] > 0.0))
                         ? 0.0 : gr[s][d];
          const double gn = sqrt(gfr[0] * gfr[0] + gfr[1] * gfr[1] + gfr[2] * gfr[2]);
          if (!(gn > 0.0)) {
            done[s] = true;
            break;
          }
          double q[3] = {gfr[0], gfr[1], gfr[2]}, al[EXT_MEM];
          for (int i = nmem[s] - 1; i >= 0; --i) {
            al[i] = RHO[s][i] * (Sm[s][i][0] * q[0] + Sm[s][i][1] * q[1] + Sm[s][i][2] * q[2]);
            for (int d = 0; d < 3; ++d) q[d] -= al[i] * Ym[s][i][d];
          }
          if (nmem[s] > 0) {
            const int l = nmem[s] - 1;
            const double sy = Sm[s][l][0] * Ym[s][l][0] + Sm[s][l][1] * Ym[s][l][1] + Sm[s][l][2] * Ym[s][l][2];
            const double yy = Ym[s][l][0] * Ym[s][l][0] + Ym[s][l][1] * Ym[s][l][1] + Ym[s][l][2] * Ym[s][l][2];
            for (int d = 0; d < 3; ++d) q[d] *= sy / yy;
          }
          for (int i = 0; i < nmem[s]; ++i) {
            const double be = RHO[s][i] * (Ym[s][i][0] * q[0] + Ym[s][i][1] * q[1] + Ym[s][i][2] * q[2]);
            for (int d = 0; d < 3; ++d) q[d] += Sm[s][i][d] * (al[i] - be);
          }
          for (int d = 0; d < 3; ++d) dir[s][d] = gfr[d] == 0.0 ? 0.0 : q[d];
          const double slope = gr[s][0] * dir[s][0] + gr[s][1] * dir[s][1] + gr[s][2] * dir[s][2];
          if (!(slope > 0.0)) {          // not an ascent direction: reset to the gradient
            nmem[s] = 0;
            for (int d = 0; d < 3; ++d) dir[s][d] = gfr[d];
          }
          dn[s] = sqrt(dir[s][0] * dir[s][0] + dir[s][1] * dir[s][1] + dir[s][2] * dir[s][2]);
          t[s] = nmem[s] == 0 ? step[s] / dn[s] : 1.0;
          if (t[s] * dn[s] > smax[s]) t[s] = smax[s] / dn[s];
          need_dir[s] = false;
        }
        if (t[s] * dn[s] < 1e-12 * smax[s]) {   // step collapsed
          if (nmem[s] > 0) {
            nmem[s] = 0;
            need_dir[s] = true;
            continue;
          }
          done[s] = true;
          break;
        }
        for (int d = 0; d < 3; ++d) {
          const double v = x[s][d] + t[s] * dir[s][d];
          xn[s][d] = v < blo[s][d] ? blo[s][d] : (v > bhi[s][d] ? bhi[s][d] : v);
        }
        break;
      }
    }
    if (done[0] && done[1]) break;
    if (bk[0] == bk[1]) {
      eval_f_grad(a, bk[0], xn, 2, sK, sV, f, gf);
    } else {
      double xa[2][3] = {{xn[0][0], xn[0][1], xn[0][2]}, {0, 0, 0}};
      double xb[2][3] = {{xn[1][0], xn[1][1], xn[1][2]}, {0, 0, 0}};
      double f1[2], gf1[2][3];
      eval_f_grad(a, bk[0], xa, 1, sK, sV, f, gf);
      eval_f_grad(a, bk[1], xb, 1, sK, sV, f1, gf1);
      f[1] = f1[0];
      for (int d = 0; d < 3; ++d) gf[1][d] = gf1[0][d];
    }
    for (int s = 0; s < 2; ++s) {
      if (done[s]) continue;
      const double Ft = sg[s] * f[s];
      double gt[3];
      for (int d = 0; d < 3; ++d) gt[d] = sg[s] * gf[s][d];
      const double gdx =
          gr[s][0] * (xn[s][0] - x[s][0]) + gr[s][1] * (xn[s][1] - x[s][1]) + gr[s][2] * (xn[s][2] - x[s][2]);
      if (Ft > F[s] && Ft >= F[s] + 1e-4 * gdx) {
        double sv[3], yv[3];
        for (int d = 0; d < 3; ++d) {
          sv[d] = xn[s][d] - x[s][d];
          yv[d] = gr[s][d] - gt[d];
        }
        const double sy = sv[0] * yv[0] + sv[1] * yv[1] + sv[2] * yv[2];
        const double ss = sqrt(sv[0] * sv[0] + sv[1] * sv[1] + sv[2] * sv[2]);
        const double ys = sqrt(yv[0] * yv[0] + yv[1] * yv[1] + yv[2] * yv[2]);
        if (sy > 1e-12 * ss * ys) {
          if (nmem[s] == EXT_MEM) {
            for (int i = 1; i < EXT_MEM; ++i) {
              for (int d = 0; d < 3; ++d) {
                Sm[s][i - 1][d] = Sm[s][i][d];
                Ym[s][i - 1][d] = Ym[s][i][d];
              }
              RHO[s][i - 1] = RHO[s][i];
            }
            --nmem[s];
          }
          for (int d = 0; d < 3; ++d) {
            Sm[s][nmem[s]][d] = sv[d];
            Ym[s][nmem[s]][d] = yv[d];
          }
          RHO[s][nmem[s]] = 1.0 / sy;
          ++nmem[s];
        }
        F[s] = Ft;
        for (int d = 0; d < 3; ++d) {
          x[s][d] = xn[s][d];
          gr[s][d] = gt[d];
        }
        need_dir[s] = true;
      } else {
        t[s] *= 0.5;
      }
    }
  }
  if ((threadIdx.x & 31) != 0) return;
  const double zmax = fmax(ext_z[2 * n], F[0]);
  const double zmin = fmin(ext_z[2 * n + 1], -F[1]);
  // U of Eq. 4 (same arithmetic as k_node_bound)
  double d = (double)(vmax[0] - base[0] + 1) * (double)(vmax[1] - base[1] + 1) * (double)(vmax[2] - base[2] + 1);
  double q_lo = 0.5 * erfc(-zmax), q_hi = 0.5 * erfc(zmin);
  double U;
  if (cs == 2) {
    U = -expm1(d * log1p(-q_lo));
  } else if (cs == 3) {
    U = -expm1(d * log1p(-q_hi));
  } else {
    U = -expm1(d * log1p(-q_lo)) - exp(d * log1p(-q_hi));
    U = U < 0.0 ? 0.0 : (U > 1.0 ? 1.0 : U);
  }
  nU[n] = U;
  nref[n] = U > a.alpha ? 1 : 0;
}

cudaError_t launch_node_extreme(Ctx& c, int level, const uint64_t* front, int64_t nF, double theta, double alpha,
                                const int8_t* ncase, int8_t* nref, double* nU, const double* ext_z,
                                const int64_t* ext_v) {
  if (nF <= 0) return cudaSuccess;
  ExtArgs a;
  a.kp = c.kp;
  a.g = c.g;
  a.k = c.k;
  a.ks = c.k + ((4 - c.k % 16) + 16) % 16;
  a.bucket_log2 = c.opts.bucket_log2;
  a.iters = c.opts.extreme_iters;
  a.bstride = c.bstride;
  a.la = la_size(c.k);
  a.bdata = c.bdata.as<double>();
  a.theta = theta;
  a.alpha = alpha;
  a.var_floor = 1e-12 * c.kp.var;
  // warp per node; as many warps per CTA (<= 8) as their K/V buffers fit in shared memory
  static const size_t static_smem = [] {
    cudaFuncAttributes at{};
    if (cudaFuncGetAttributes(&at, k_node_extreme) != cudaSuccess) {
      cudaGetLastError();
      return (size_t)4096;
    }
    return (size_t)at.sharedSizeBytes;
  }();
  const size_t per_warp = sizeof(double) * (8 * (size_t)a.ks + (c.k > 128 ? 1024 : 0));
  const size_t cap = 227 * 1024 - static_smem - 512;
  const int warps = (int)std::min<size_t>(8, cap / per_warp);
  if (warps < 1) return cudaErrorInvalidConfiguration;
  size_t smem = per_warp * warps;
  cudaError_t e = cudaFuncSetAttribute(k_node_extreme, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  unsigned grid = (unsigned)((nF + warps - 1) / warps);
  k_node_extreme<<<grid, 32 * warps, smem, c.stream>>>(a, level, front, nF, ncase, nref, nU, ext_z, ext_v);
  ++c.n_launch;
  return cudaGetLastError();
}

}  // namespace lcp
