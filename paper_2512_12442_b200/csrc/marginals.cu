// marginals.cu -- bucket-tiled local-GP posterior kernels.
//
// Eq. 1 on the bucket's local GP (R1, R2): for query points
// q_1..q_8 sharing bucket B with observations S_B, factor L_B (K_y = L L^T) and
// alpha_B = K_y^-1 (y_S - m0):
//     mu_c    = m0 + sum_j K(x_j, q_c) alpha_j
//     V       = L^-1 K_{S,q}            (k x 8, triangular mat-mat)
//     Sigma   = K_qq - V^T V
// One warp handles 8 queries: the 8 corners of a cell (leaf pass, a7) or 8
// independent points (vertex / observation marginals, a4-a5).  A CTA stages the
// bucket block [L^-1 | alpha | X_S] into shared memory once and all its warps
// reuse it; work lists are grouped by bucket (scan.cu) so restaging is rare.
#include <algorithm>

#include "ctx.h"

namespace lcp {

constexpr int TILE_WARPS_MAX = 16;
constexpr int ROWS_PER_GROUP = 128;   // 4 row blocks of 32 per lane pass

struct TileArgs {
  KernParams kp;
  Geom g;
  int k;
  int staged;            // L^-1 staged in shared memory
  int64_t bstride;       // doubles per bucket block
  const double* bdata;   // [L^-1 A-fragments (la_size(k)) | alpha | x | y | z] per bucket
  double kcc[36];        // prior covariance of the 8 cell corners (packed lower, row-major pairs)
  int64_t la;            // doubles of the L^-1 A-fragment block (la_size(k))
  int ks;                // row stride of the per-warp K buffer sK[c][j] (ks = 4 mod 16: conflict-free)
  double var_floor;      // 1e-12 sigma_f^2
  double var_err;        // -1e-8 sigma_f^2
};

// all threads copy n doubles (16-byte aligned) global -> shared
__device__ __forceinline__ void stage_copy(double* dst, const double* __restrict__ src, int64_t n) {
  const double2* s2 = reinterpret_cast<const double2*>(src);
  double2* d2 = reinterpret_cast<double2*>(dst);
  int64_t n2 = n >> 1;
  for (int64_t i = threadIdx.x; i < n2; i += blockDim.x) d2[i] = __ldg(s2 + i);
  if ((n & 1) && threadIdx.x == 0) dst[n - 1] = __ldg(src + n - 1);
}

__device__ __forceinline__ void dmma884(double a, double b, double& d0, double& d1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// V rows [row0, row0 + 128) of V = L^-1 K (8 columns) on the FP64 tensor cores
// (DMMA.8x8x4).  Fragment layout (probe tools/probes/dmma_layout.cu): A[lane>>2][lane&3],
// B[lane&3][lane>>2], C[lane>>2][2 (lane&3) + {0,1}].  acc[t] holds
// V[row0 + 8 t + (lane>>2)][2 (lane&3) + {0,1}].
__device__ __forceinline__ void v_group_dmma(const double* __restrict__ LA, int k, int ks, int row0,
                                             const double* __restrict__ sK, double (&acc)[16][2], int lane) {
#pragma unroll
  for (int t = 0; t < 16; ++t) acc[t][0] = acc[t][1] = 0.0;
  const int lr = lane >> 2, lc = lane & 3;
  const int nrows = min(ROWS_PER_GROUP, k - row0);
  const int nrt = (nrows + 7) >> 3;
  const int rt0 = row0 >> 3;
  const int jend = row0 + 8 * nrt;
  for (int j = 0; j < jend; j += 4) {
    const int jj = j + lc, js = j >> 2;
    const double b = jj < k ? sK[lr * ks + jj] : 0.0;
    const int rt_lo = j < row0 ? 0 : ((j - row0) >> 3);
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      if (t < rt_lo || t >= nrt) continue;   // warp-uniform: zero block of L^-1
      dmma884(LA[la_block(rt0 + t, js) + lane], b, acc[t][0], acc[t][1]);
    }
  }
}

// Warp computes, for its 8 queries (positions in sQ[8][3]):
//   mu_out  : lane c (< 8) holds mu of query c
//   diag_only: out[e] = sum_i V[i][2 (lane&3) + e]^2   (every lane)
//   full     : out[e] = D[lane>>2][2 (lane&3) + e],  D = V^T V (8x8)
__device__ __forceinline__ void warp_local_posterior(const TileArgs& a, const double* __restrict__ Linv,
                                                     const double* __restrict__ alpha,
                                                     const double* __restrict__ Xs,
                                                     const double* __restrict__ sQ, double* sK, double* sV,
                                                     bool diag_only, double& mu_out, double (&out)[2]) {
  const int k = a.k;
  const int lane = threadIdx.x & 31;
  const int lr = lane >> 2, lc = lane & 3;
  const int ks = a.ks;
  // 1. K[c][j] = k(x_j, q_c)  (query-major: lanes over j store conflict-free)
  for (int j = lane; j < k; j += 32) {
    double xj = Xs[j], yj = Xs[k + j], zj = Xs[2 * k + j];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double r2 = kern_r2(a.kp, xj - sQ[3 * c], yj - sQ[3 * c + 1], zj - sQ[3 * c + 2]);
      sK[c * ks + j] = kern_from_r2(a.kp, r2);
    }
  }
  __syncwarp();
  // 2. mu_c = m0 + sum_j K[c][j] alpha_j   (lane: c = lane & 7, part = lane >> 3)
  {
    int c = lane & 7, part = lane >> 3;
    double s = 0.0;
    for (int j = part; j < k; j += 4) s = fma(sK[c * ks + j], alpha[j], s);
    s += __shfl_xor_sync(0xffffffffu, s, 8);
    s += __shfl_xor_sync(0xffffffffu, s, 16);
    mu_out = a.kp.m0 + s;
  }
  // 3. V = L^-1 K by row groups of 128 (DMMA); 4. diag or V^T V (DMMA)
  double o0 = 0.0, o1 = 0.0;
  const bool single = k <= ROWS_PER_GROUP;
  for (int row0 = 0; row0 < k; row0 += ROWS_PER_GROUP) {
    double acc[16][2];
    v_group_dmma(Linv, k, ks, row0, sK, acc, lane);
    const int nrows = min(ROWS_PER_GROUP, k - row0);
    if (diag_only) {
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        o0 = fma(acc[t][0], acc[t][0], o0);
        o1 = fma(acc[t][1], acc[t][1], o1);
      }
    } else {
      double* dst = single ? sK : sV;   // single group: K is dead, reuse its buffer
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
        dmma884(v, v, o0, o1);
      }
      __syncwarp();
    }
  }
  if (diag_only) {
    // rows were spread over lr: reduce across lanes with the same (lane & 3)
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      o0 += __shfl_xor_sync(0xffffffffu, o0, o);
      o1 += __shfl_xor_sync(0xffffffffu, o1, o);
    }
  }
  out[0] = o0;
  out[1] = o1;
}

__device__ __forceinline__ int item_bucket(const TileArgs& a, int mode, int64_t item, const double* pts,
                                           const int32_t* bkt_sorted, int64_t q) {
  if (bkt_sorted) return bkt_sorted[q];
  if (mode == Q_VERTEX) return vertex_bucket(a.g, item);
  return cell_bucket(a.g, item);
}

// Generic tile loop: CTA handles sorted positions [t0, t1) (t1 - t0 <= TILE_MAX);
// runs of equal bucket are found in parallel (ballot + warp-prefix compaction)
// and share one staging of the bucket block.
constexpr int TILE_MAX = 2048;

template <int STAGED, typename Body>
__device__ __forceinline__ void tile_loop(const TileArgs& a, int64_t t0, int64_t t1, double* smem,
                                          const int32_t* __restrict__ runb, Body body) {
  __shared__ int s_starts[TILE_MAX + 1];
  __shared__ int s_wcnt[33];
  __shared__ int s_nruns;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int n = (int)(t1 - t0);
  if (tid == 0) s_nruns = 0;
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + tid;
    const bool f = i < n && (i == 0 || runb[t0 + i] != runb[t0 + i - 1]);
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_wcnt[wid] = __popc(bal);
    __syncthreads();
    if (wid == 0) {
      int v = lane < nw ? s_wcnt[lane] : 0, x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane < nw) s_wcnt[lane] = x - v;
      if (lane == 31) s_wcnt[32] = x;
    }
    __syncthreads();
    if (f) s_starts[s_nruns + s_wcnt[wid] + __popc(bal & ((1u << lane) - 1u))] = i;
    __syncthreads();
    if (tid == 0) s_nruns += s_wcnt[32];
    __syncthreads();
  }
  const int nruns = s_nruns;
  if (tid == 0) s_starts[nruns] = n;
  __syncthreads();
  const int64_t blk = a.bstride;
  int staged_bucket = -1;
  for (int r = 0; r < nruns; ++r) {
    const int64_t q = t0 + s_starts[r], qe = t0 + s_starts[r + 1];
    const int b = runb[q];
    if (b != staged_bucket) {
      const double* src = a.bdata + (int64_t)b * blk;
      if (STAGED) stage_copy(smem, src, blk);
      else stage_copy(smem, src + a.la, 4 * (int64_t)a.k);
      staged_bucket = b;
    }
    __syncthreads();
    // STAGED is a template parameter so that Linv is a known shared (or global) pointer
    const double* Linv = STAGED ? smem : a.bdata + (int64_t)b * blk;
    const double* tail = STAGED ? smem + a.la : smem;
    body(b, q, qe, Linv, tail, tail + a.k);
    __syncthreads();
  }
}

// ---------------------------------------------------------------- a4 / a5
// items_sorted[q]: vertex id (Q_VERTEX), observation index (Q_OBS) or point
// index (Q_POINT); bkt_sorted[q]: its bucket.  Output indexed by the item
// (vertex cache slot, observation, point).
template <int STAGED>
__global__ void __launch_bounds__(512) k_marginals(TileArgs a, int mode, const int64_t* __restrict__ items,
                                                   const int32_t* __restrict__ bkt_sorted, int64_t n,
                                                   const int64_t* __restrict__ n_dev, int tile,
                                                   const double* __restrict__ pts, double* __restrict__ out_mu,
                                                   double* __restrict__ out_sd, int write_var,
                                                   double2* __restrict__ vcache, uint8_t* __restrict__ vstate,
                                                   int* __restrict__ derr) {
  extern __shared__ double smem[];
  if (n_dev) n = *n_dev;
  int64_t t0 = (int64_t)blockIdx.x * tile;
  if (t0 >= n) return;
  int64_t t1 = min(n, t0 + tile);
  const int warps = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = a.k;
  int64_t head = STAGED ? a.bstride : 4 * (int64_t)k;
  head = (head + 1) & ~1ll;
  const int64_t per_warp = 8 * (int64_t)a.ks + (k > ROWS_PER_GROUP ? 8 * ROWS_PER_GROUP : 0) + 24;
  double* wbuf = smem + head + wid * per_warp;
  double* sK = wbuf;
  double* sV = wbuf + 8 * a.ks;
  double* sQ = wbuf + per_warp - 24;
  const Geom& g = a.g;
  tile_loop<STAGED>(a, t0, t1, smem, bkt_sorted, [&](int b, int64_t q0, int64_t q1, const double* Linv,
                                              const double* alpha, const double* Xs) {
    for (int64_t base = q0 + 8 * wid; base < q1; base += 8 * warps) {
      int nq = (int)min((int64_t)8, q1 - base);
      if (lane < 8) {
        int64_t it = items[base + (lane < nq ? lane : 0)];
        double x, y, z;
        if (mode == Q_VERTEX) {
          int i, j, kk;
          vertex_ijk(g, it, i, j, kk);
          x = vpos(g, 0, i); y = vpos(g, 1, j); z = vpos(g, 2, kk);
        } else {
          x = pts[3 * it]; y = pts[3 * it + 1]; z = pts[3 * it + 2];
        }
        sQ[3 * lane] = x; sQ[3 * lane + 1] = y; sQ[3 * lane + 2] = z;
      }
      __syncwarp();
      double mu, pr[2];
      warp_local_posterior(a, Linv, alpha, Xs, sQ, sK, sV, true, mu, pr);
      // query c's sum of squares sits in lane c >> 1, element c & 1
      const double sq0 = __shfl_sync(0xffffffffu, pr[0], lane >> 1);
      const double sq1 = __shfl_sync(0xffffffffu, pr[1], lane >> 1);
      if (lane < nq) {
        int64_t it = items[base + lane];
        double var = a.kp.var - ((lane & 1) ? sq1 : sq0);   // k(q,q) = sigma_f^2 for both kernels
        if (var < a.var_err) atomicOr(derr, DERR_NUMERIC);
        double vf = var > a.var_floor ? var : a.var_floor;
        if (mode == Q_VERTEX) {
          vcache[it] = make_double2(mu, 1.0 / (sqrt(vf) * SQRT2));   // (mu, 1 / (sigma sqrt 2))
        } else {
          out_mu[it] = mu;
          out_sd[it] = write_var ? var : sqrt(vf);
        }
      }
      __syncwarp();
    }
  });
}

// ------------------------------------------------------------------- a7
// post[q] (44 doubles): mu[8] then Sigma packed lower (pair p = c(c+1)/2 + d).
template <int STAGED>
__global__ void __launch_bounds__(512) k_cell_posterior(TileArgs a, const int64_t* __restrict__ cells,
                                                        const int64_t* __restrict__ perm,
                                                        const int32_t* __restrict__ bkt_sorted, int64_t n,
                                                        int tile, double* __restrict__ post,
                                                        int* __restrict__ derr) {
  extern __shared__ double smem[];
  int64_t t0 = (int64_t)blockIdx.x * tile;
  if (t0 >= n) return;
  int64_t t1 = min(n, t0 + tile);
  const int warps = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = a.k;
  int64_t head = STAGED ? a.bstride : 4 * (int64_t)k;
  head = (head + 1) & ~1ll;
  const int64_t per_warp = 8 * (int64_t)a.ks + (k > ROWS_PER_GROUP ? 8 * ROWS_PER_GROUP : 0) + 24;
  double* wbuf = smem + head + wid * per_warp;
  double* sK = wbuf;
  double* sV = wbuf + 8 * a.ks;
  double* sQ = wbuf + per_warp - 24;
  const Geom& g = a.g;
  tile_loop<STAGED>(a, t0, t1, smem, bkt_sorted, [&](int b, int64_t q0, int64_t q1, const double* Linv,
                                              const double* alpha, const double* Xs) {
    for (int64_t q = q0 + wid; q < q1; q += warps) {
      int64_t slot = perm ? perm[q] : q;
      int64_t cell = cells[slot];
      int ci, cj, ck;
      cell_ijk(g, cell, ci, cj, ck);
      if (lane < 8) {
        sQ[3 * lane] = vpos(g, 0, ci + (lane & 1));
        sQ[3 * lane + 1] = vpos(g, 1, cj + ((lane >> 1) & 1));
        sQ[3 * lane + 2] = vpos(g, 2, ck + (lane >> 2));
      }
      __syncwarp();
      double mu, pr[2];
      warp_local_posterior(a, Linv, alpha, Xs, sQ, sK, sV, false, mu, pr);
      double* rec = post + 44 * slot;
      if (lane < 8) rec[lane] = mu;
      // lane holds D[r][c] for r = lane >> 2, c = 2 (lane & 3) + e; keep c <= r
      const int r = lane >> 2;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = 2 * (lane & 3) + e;
        if (cc <= r) {
          const int p = r * (r + 1) / 2 + cc;
          const double sv = a.kcc[p] - pr[e];
          rec[8 + p] = sv;
          if (cc == r && sv < a.var_err) atomicOr(derr, DERR_NUMERIC);
        }
      }
      __syncwarp();
    }
  });
}

// R17 (BASELINE c2 "FP32 posterior"): the same posterior with the cross-covariance,
// the solve V = L^-1 K and Sigma = K_cc - V^T V in FP32 (CUDA-core FFMA) from the
// FP64-built bucket factor (cast on load); mu and Sigma are stored widened to FP64
// and the 8x8 Cholesky stays FP64 (k_chol8).  Warp per cell, k <= 128.  The mean's
// k-term dot product K_*^T alpha accumulates in FP64 (8 DFMA per observation, FP64
// alpha): its error is then the FP32 rounding of the kernel values alone,
// ~eps32 sum_j |k_j alpha_j|, which a large sum |alpha| (ill-conditioned K_SS)
// still lifts above 1e-4 sigma_f -- the FP32 bound the tests state (DESIGN R17).
template <int STAGED>
__global__ void __launch_bounds__(512) k_cell_posterior_f32(TileArgs a, const int64_t* __restrict__ cells,
                                                            const int64_t* __restrict__ perm,
                                                            const int32_t* __restrict__ bkt_sorted, int64_t n,
                                                            int tile, double* __restrict__ post,
                                                            int* __restrict__ derr) {
  extern __shared__ double smem[];
  int64_t t0 = (int64_t)blockIdx.x * tile;
  if (t0 >= n) return;
  int64_t t1 = min(n, t0 + tile);
  const int warps = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = a.k;
  int64_t head = STAGED ? a.bstride : 4 * (int64_t)k;
  head = (head + 1) & ~1ll;
  const int64_t per_warp = 8 * (int64_t)a.ks + (k > ROWS_PER_GROUP ? 8 * ROWS_PER_GROUP : 0) + 24;
  float* sKf = reinterpret_cast<float*>(smem + head + wid * per_warp);   // [j][8] floats
  const Geom& g = a.g;
  tile_loop<STAGED>(a, t0, t1, smem, bkt_sorted, [&](int b, int64_t q0, int64_t q1, const double* LA,
                                              const double* alpha, const double* Xs) {
    for (int64_t q = q0 + wid; q < q1; q += warps) {
      int64_t slot = perm ? perm[q] : q;
      int ci, cj, ck;
      cell_ijk(g, cells[slot], ci, cj, ck);
      float qx[8][3];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        qx[c][0] = (float)vpos(g, 0, ci + (c & 1));
        qx[c][1] = (float)vpos(g, 1, cj + ((c >> 1) & 1));
        qx[c][2] = (float)vpos(g, 2, ck + (c >> 2));
      }
      const float var_f = (float)a.kp.var;
      const float il[3] = {(float)a.kp.inv_ls[0], (float)a.kp.inv_ls[1], (float)a.kp.inv_ls[2]};
      double mu_p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int j = lane; j < k; j += 32) {
        const float xj = (float)Xs[j], yj = (float)Xs[k + j], zj = (float)Xs[2 * k + j];
        const double al = alpha[j];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float tx = (xj - qx[c][0]) * il[0], ty = (yj - qx[c][1]) * il[1], tz = (zj - qx[c][2]) * il[2];
          // clamp: the far padding dummies of beta-box sets (R28) overflow FP32 squares, and
          // Matern's inf * 0 would give NaN; at 1e30 both kernels are exactly 0 in FP32
          float r2 = fminf(tx * tx + ty * ty + tz * tz, 1e30f), kv;
          if (a.kp.kind == LCP_K_SE) {
            kv = var_f * expf(-0.5f * r2);
          } else {
            float r = sqrtf(r2), s5 = 2.2360679775f * r;
            kv = var_f * (1.0f + s5 + (5.0f / 3.0f) * r2) * expf(-s5);
          }
          sKf[8 * j + c] = kv;
          mu_p[c] = fma((double)kv, al, mu_p[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) mu_p[c] = warp_sum(mu_p[c]);
      __syncwarp();
      // V rows i = lane + 32 rb; pair partial sums of V^T V
      float pp[36];
#pragma unroll
      for (int p = 0; p < 36; ++p) pp[p] = 0.0f;
#pragma unroll
      for (int rb = 0; rb < 4; ++rb) {
        const int i = lane + 32 * rb;
        if (32 * rb >= k) break;
        float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (i < k) {
          const int rt = i >> 3, ri = i & 7;
          for (int j = 0; j <= i; ++j) {
            const float l = (float)LA[la_block(rt, j >> 2) + 4 * ri + (j & 3)];
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = fmaf(l, sKf[8 * j + c], v[c]);
          }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
          for (int d = 0; d <= c; ++d) pp[c * (c + 1) / 2 + d] = fmaf(v[c], v[d], pp[c * (c + 1) / 2 + d]);
      }
#pragma unroll
      for (int p = 0; p < 36; ++p) pp[p] = warp_sum(pp[p]);
      double* rec = post + 44 * slot;
      if (lane < 8) {
        double muv = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) muv = lane == c ? mu_p[c] : muv;
        rec[lane] = a.kp.m0 + muv;
      }
      if (lane == 0) {
#pragma unroll
        for (int p = 0; p < 36; ++p) {
          const double sv = (double)((float)a.kcc[p] - pp[p]);
          rec[8 + p] = sv;
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (rec[8 + c * (c + 3) / 2] < a.var_err) atomicOr(derr, DERR_NUMERIC);
      }
      __syncwarp();
    }
  });
}

static TileArgs make_tile_args(Ctx& c) {
  TileArgs a;
  a.kp = c.kp;
  a.g = c.g;
  a.k = c.k;
  a.bstride = c.bstride;
  a.bdata = c.bdata.as<double>();
  for (int p = 0; p < 36; ++p) a.kcc[p] = c.kcc[p];
  a.var_floor = 1e-12 * c.kp.var;
  a.la = la_size(c.k);
  a.ks = c.k + ((4 - c.k % 16) + 16) % 16;
  a.var_err = -1e-8 * c.kp.var;
  a.staged = 0;
  return a;
}

// shared-memory plan: staged bucket block (if it fits) + W per-warp buffers
// static shared memory of the tile kernels (tile_loop's run table): the dynamic
// cap is 227 KB minus this (a launch over the opt-in limit fails with "invalid argument")
static size_t tile_static_smem() {
  static const size_t v = [] {
    size_t mx = 0;
    const void* fs[] = {(const void*)k_marginals<0>, (const void*)k_marginals<1>,
                        (const void*)k_cell_posterior<0>, (const void*)k_cell_posterior<1>,
                        (const void*)k_cell_posterior_f32<0>, (const void*)k_cell_posterior_f32<1>};
    for (const void* f : fs) {
      cudaFuncAttributes at{};
      if (cudaFuncGetAttributes(&at, f) == cudaSuccess) mx = std::max(mx, (size_t)at.sharedSizeBytes);
    }
    cudaGetLastError();
    return mx;
  }();
  return v;
}

static void plan_tile(const Ctx& c, int& staged, int& warps, size_t& smem) {
  const size_t cap = std::min<size_t>(220 * 1024, 227 * 1024 - tile_static_smem() - 512);
  int64_t k = c.k;
  const int64_t ks = k + ((4 - k % 16) + 16) % 16;
  size_t per_warp = sizeof(double) * (8 * ks + (k > ROWS_PER_GROUP ? 8 * ROWS_PER_GROUP : 0) + 24);
  size_t head_staged = sizeof(double) * ((c.bstride + 1) & ~1ll);
  size_t head_tail = sizeof(double) * (4 * k + 1);
  staged = 0;
  warps = 0;
  for (int w = TILE_WARPS_MAX; w >= 4; w -= 4) {
    if (head_staged + w * per_warp <= cap) { staged = 1; warps = w; break; }
  }
  if (!staged) {
    for (int w = TILE_WARPS_MAX; w >= 1; --w)
      if (head_tail + w * per_warp <= cap) { warps = w; break; }
    smem = head_tail + warps * per_warp;
  } else {
    smem = head_staged + warps * per_warp;
  }
}

cudaError_t launch_marginals(Ctx& c, int mode, const int64_t* items_sorted, const int32_t* bkt_sorted,
                             int64_t n, const double* points, double* out_mu, double* out_sd,
                             int write_var, const int64_t* n_dev) {
  if (n <= 0) return cudaSuccess;
  TileArgs a = make_tile_args(c);
  int staged, warps;
  size_t smem;
  plan_tile(c, staged, warps, smem);
  if (warps == 0) return cudaErrorInvalidConfiguration;
  int tile = std::min(8 * warps * 8, TILE_MAX);
  if (n_dev == nullptr && n < 8 * (int64_t)c.g.nbuckets && c.g.nbuckets > 1) {
    // sparse items (few per bucket, e.g. the observation marginals of a fine bucket
    // grid): staging a whole bucket block per item would dominate, so L^-1 is read
    // straight from global memory by small CTAs (2 warps, 16 items each)
    const int64_t k = c.k;
    const int64_t ks = k + ((4 - k % 16) + 16) % 16;
    const size_t per_warp = sizeof(double) * (8 * ks + (k > ROWS_PER_GROUP ? 8 * ROWS_PER_GROUP : 0) + 24);
    staged = 0;
    warps = 2;
    smem = sizeof(double) * (4 * k + 1) + warps * per_warp;
    tile = 16;
  }
  a.staged = staged;
  auto kern = staged ? k_marginals<1> : k_marginals<0>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned grid = (unsigned)((n + tile - 1) / tile);
  kern<<<grid, 32 * warps, smem, c.stream>>>(a, mode, items_sorted, bkt_sorted, n, n_dev, tile, points,
                                                    out_mu, out_sd, write_var, c.vcache.as<double2>(),
                                                    c.vstate.as<uint8_t>(), c.derr.as<int>());
  ++c.n_launch;
  return cudaGetLastError();
}

cudaError_t launch_cell_posterior(Ctx& c, const int64_t* cells, const int64_t* perm,
                                  const int32_t* bkt_sorted, int64_t n, double* post) {
  if (c.opts.precision == LCP_FP32 && c.k <= 128) {
    if (n <= 0) return cudaSuccess;
    TileArgs a = make_tile_args(c);
    int staged, warps;
    size_t smem;
    plan_tile(c, staged, warps, smem);
    if (warps == 0) return cudaErrorInvalidConfiguration;
    a.staged = staged;
    auto kf = staged ? k_cell_posterior_f32<1> : k_cell_posterior_f32<0>;
    cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int tile = warps * 16;
    unsigned grid = (unsigned)((n + tile - 1) / tile);
    kf<<<grid, 32 * warps, smem, c.stream>>>(a, cells, perm, bkt_sorted, n, tile, post,
                                                               c.derr.as<int>());
    ++c.n_launch;
    return cudaGetLastError();
  }
  if (n <= 0) return cudaSuccess;
  TileArgs a = make_tile_args(c);
  int staged, warps;
  size_t smem;
  plan_tile(c, staged, warps, smem);
  if (warps == 0) return cudaErrorInvalidConfiguration;
  a.staged = staged;
  auto kc = staged ? k_cell_posterior<1> : k_cell_posterior<0>;
  cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int tile = warps * 16;
  unsigned grid = (unsigned)((n + tile - 1) / tile);
  kc<<<grid, 32 * warps, smem, c.stream>>>(a, cells, perm, bkt_sorted, n, tile, post,
                                                         c.derr.as<int>());
  ++c.n_launch;
  return cudaGetLastError();
}

}  // namespace lcp
