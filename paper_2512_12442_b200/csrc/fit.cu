// fit.cu -- lcp_fit_local: SURVEY §8(a) rows a1-a4.
//
//  a1  k_obs_bin / group_by_bucket / k_obs_rank : point -> bucket (R3), finest
//      cell, Morton key of the finest cell, observations grouped by bucket and
//      sorted by Morton key (for the node ranges of Alg. 1 line 3).
//  a2  k_knn        : per bucket, the k nearest observations to the bucket centre
//      in the metric sum_d ((x_d - c_d) / l_d)^2, ties -> lower index (R2); exact
//      ring search over the bucket grid, brute-force fallback k_knn_brute.
//  a3  k_bucket_factor : K_y = K_SS + sigma_n^2 I, Cholesky, L^-1 and
//      alpha = K_y^-1 (y_S - m0) (Eq. 1; jitter R15).
//  a4  observation marginals (R10) via k_marginals.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "ctx.h"

namespace lcp {

constexpr int KNN_CMAX = 6144;
constexpr int KNN_THREADS = 256;
constexpr int FACT_THREADS = 256;

template <typename T>
__device__ T block_sum(T v, T* sh) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  T s = 0;
  for (int w = 0; w < nw; ++w) s += sh[w];
  return s;
}

// a1: point bucket, finest cell Morton key
__global__ void k_obs_bin(Geom g, const double* __restrict__ X, const double* __restrict__ Y, int64_t m,
                          int32_t* __restrict__ obs_bucket, uint64_t* __restrict__ obs_key, int* __restrict__ derr) {
  int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= m) return;
  if (!isfinite(Y[o]) || !isfinite(X[3 * o]) || !isfinite(X[3 * o + 1]) || !isfinite(X[3 * o + 2]))
    atomicOr(derr, DERR_INPUT);
  int bc[3], cc[3];
  for (int d = 0; d < 3; ++d) {
    double x = X[3 * o + d];
    bc[d] = point_bucket_axis(g, d, x);
    cc[d] = cell_axis(g, d, x);
  }
  obs_bucket[o] = bucket_id(g, bc[0], bc[1], bc[2]);
  obs_key[o] = morton3(cc[0], cc[1], cc[2]);
}

// DERR_INPUT if any of n values is not finite (grid-stride)
__global__ void k_check_finite(const double* __restrict__ v, int64_t n, int* __restrict__ derr) {
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(v[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(derr, DERR_INPUT);
}

// occupancy bitmaps: bit (key >> 3h) of occ_h set for every observation's finest-cell key
__global__ void k_occ_set(const uint64_t* __restrict__ key, int64_t m, int nh, uint32_t* __restrict__ o0,
                          uint32_t* __restrict__ o1, uint32_t* __restrict__ o2) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  const uint64_t kk = key[q];
  uint32_t* o[3] = {o0, o1, o2};
  for (int h = 0; h < nh; ++h) {
    const uint64_t c = kk >> (3 * h);
    atomicOr(&o[h][c >> 5], 1u << (c & 31));
  }
}

__global__ void k_bucket_ranges(const int64_t* __restrict__ gcount, const int64_t* __restrict__ gend, int nb,
                                int64_t* __restrict__ bcount, int64_t* __restrict__ bstart) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  bcount[b] = gcount[b];
  bstart[b] = gend[b] - gcount[b];
}

__global__ void k_gather_i32(const int32_t* __restrict__ src, const int64_t* __restrict__ perm, int64_t n,
                             int32_t* __restrict__ dst) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) dst[q] = src[perm[q]];
}

// a1: stable rank sort of the Morton keys (m is at most ~1e5: O(m^2 / P))
__global__ void k_obs_rank(const uint64_t* __restrict__ key, int64_t m, uint64_t* __restrict__ skey,
                           int32_t* __restrict__ sidx) {
  __shared__ uint64_t tile[1024];
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t ki = i < m ? key[i] : 0;
  int64_t rank = 0;
  for (int64_t t0 = 0; t0 < m; t0 += 1024) {
    __syncthreads();
    for (int q = threadIdx.x; q < 1024; q += blockDim.x)
      tile[q] = t0 + q < m ? key[t0 + q] : ~0ull;
    __syncthreads();
    if (i < m) {
      int n = (int)min((int64_t)1024, m - t0);
      for (int q = 0; q < n; ++q) {
        uint64_t kj = tile[q];
        rank += (kj < ki) || (kj == ki && t0 + q < i);
      }
    }
  }
  if (i < m) {
    skey[rank] = ki;
    sidx[rank] = (int32_t)i;
  }
}

// a2: exact k-NN by ring search over the bucket grid.  A ball of radius
// R_out (the metric distance from the centre to the nearest face of the
// searched box that is not the grid boundary) contains every observation
// outside the box at distance >= R_out; the k-th candidate distance strictly
// inside R_out (with a 1e-9 relative margin) proves the candidate set exact.
__global__ void __launch_bounds__(KNN_THREADS) k_knn(KernParams kp, Geom g, const double* __restrict__ X,
                                                     int64_t m, int k, const int64_t* __restrict__ bstart,
                                                     const int64_t* __restrict__ bcount,
                                                     const int64_t* __restrict__ obs_by_bucket,
                                                     int32_t* __restrict__ S, int* __restrict__ fail_list,
                                                     int* __restrict__ n_fail, int r0, int b0) {
  extern __shared__ unsigned char sm_raw[];
  double* cd2 = reinterpret_cast<double*>(sm_raw);
  int32_t* cidx = reinterpret_cast<int32_t*>(cd2 + KNN_CMAX);
  int32_t* sel = cidx + KNN_CMAX;
  __shared__ long long s_red[32];
  __shared__ int s_n;
  __shared__ double s_d2k;
  const int b = b0 + blockIdx.x;
  int32_t* Sb = S + (int64_t)b * k;
  if ((int64_t)k >= m) {
    for (int a = threadIdx.x; a < k; a += blockDim.x) Sb[a] = a;
    return;
  }
  int bc[3] = {b % g.nb[0], (b / g.nb[0]) % g.nb[1], b / (g.nb[0] * g.nb[1])};
  double c[3];
  for (int d = 0; d < 3; ++d) c[d] = __dadd_rn(g.lo[d], __dmul_rn((double)bc[d] + 0.5, g.sB[d]));
  for (int r = r0;; ++r) {
    __syncthreads();
    int lo[3], hi[3], ext[3];
    bool full = true;
    for (int d = 0; d < 3; ++d) {
      lo[d] = max(bc[d] - r, 0);
      hi[d] = min(bc[d] + r, g.nb[d] - 1);
      ext[d] = hi[d] - lo[d] + 1;
      full = full && lo[d] == 0 && hi[d] == g.nb[d] - 1;
    }
    int64_t nbox = (int64_t)ext[0] * ext[1] * ext[2];
    long long cnt = 0;
    for (int64_t t = threadIdx.x; t < nbox; t += blockDim.x) {
      int ix = lo[0] + (int)(t % ext[0]), iy = lo[1] + (int)((t / ext[0]) % ext[1]),
          iz = lo[2] + (int)(t / ((int64_t)ext[0] * ext[1]));
      cnt += bcount[bucket_id(g, ix, iy, iz)];
    }
    cnt = block_sum(cnt, s_red);
    if (cnt > KNN_CMAX) {
      if (threadIdx.x == 0) fail_list[atomicAdd(n_fail, 1)] = b;
      return;
    }
    if (cnt < k && !full) continue;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int64_t t = threadIdx.x; t < nbox; t += blockDim.x) {
      int ix = lo[0] + (int)(t % ext[0]), iy = lo[1] + (int)((t / ext[0]) % ext[1]),
          iz = lo[2] + (int)(t / ((int64_t)ext[0] * ext[1]));
      int id = bucket_id(g, ix, iy, iz);
      int64_t st = bstart[id], n = bcount[id];
      for (int64_t q = 0; q < n; ++q) {
        int64_t o = obs_by_bucket[st + q];
        int pos = atomicAdd(&s_n, 1);
        cidx[pos] = (int32_t)o;
        cd2[pos] = knn_d2(kp, X + 3 * o, c);
      }
    }
    __syncthreads();
    const int n = s_n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double di = cd2[i];
      int32_t ii = cidx[i];
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        double dj = cd2[j];
        rank += (dj < di) || (dj == di && cidx[j] < ii);
      }
      if (rank < k) sel[rank] = ii;
      if (rank == k - 1) s_d2k = di;
    }
    __syncthreads();
    if (!full) {
      double rout2 = INFINITY;
      for (int d = 0; d < 3; ++d) {
        if (lo[d] > 0 || hi[d] < g.nb[d] - 1) {
          double f = __dmul_rn(__dmul_rn((double)r + 0.5, g.sB[d]), kp.inv_ls[d]);
          rout2 = fmin(rout2, f * f);
        }
      }
      if (!(s_d2k < rout2 * (1.0 - 1e-9))) continue;
    }
    for (int a = threadIdx.x; a < k; a += blockDim.x) {
      int32_t v = sel[a];
      int rk = 0;
      for (int q = 0; q < k; ++q) rk += sel[q] < v;
      Sb[rk] = v;
    }
    return;
  }
}

// a2 fallback: running top-k over all observations in chunks (exact, slow)
__global__ void __launch_bounds__(KNN_THREADS) k_knn_brute(KernParams kp, Geom g, const double* __restrict__ X,
                                                           int64_t m, int k, const int* __restrict__ list,
                                                           int32_t* __restrict__ S) {
  extern __shared__ unsigned char sm_raw[];
  double* cd2 = reinterpret_cast<double*>(sm_raw);
  int32_t* cidx = reinterpret_cast<int32_t*>(cd2 + KNN_CMAX);
  int32_t* sel = cidx + KNN_CMAX;
  double* seld = reinterpret_cast<double*>(sel + ((k + 1) & ~1));
  const int b = list[blockIdx.x];
  int bc[3] = {b % g.nb[0], (b / g.nb[0]) % g.nb[1], b / (g.nb[0] * g.nb[1])};
  double c[3];
  for (int d = 0; d < 3; ++d) c[d] = __dadd_rn(g.lo[d], __dmul_rn((double)bc[d] + 0.5, g.sB[d]));
  int ntop = 0;
  const int chunk = KNN_CMAX - k;
  for (int64_t s0 = 0; s0 < m; s0 += chunk) {
    int nn = (int)min((int64_t)chunk, m - s0);
    for (int t = threadIdx.x; t < nn; t += blockDim.x) {
      cidx[ntop + t] = (int32_t)(s0 + t);
      cd2[ntop + t] = knn_d2(kp, X + 3 * (s0 + t), c);
    }
    __syncthreads();
    int n = ntop + nn;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double di = cd2[i];
      int32_t ii = cidx[i];
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        double dj = cd2[j];
        rank += (dj < di) || (dj == di && cidx[j] < ii);
      }
      if (rank < k) { sel[rank] = ii; seld[rank] = di; }
    }
    __syncthreads();
    ntop = min(k, n);
    for (int t = threadIdx.x; t < ntop; t += blockDim.x) { cidx[t] = sel[t]; cd2[t] = seld[t]; }
    __syncthreads();
  }
  int32_t* Sb = S + (int64_t)b * k;
  for (int a = threadIdx.x; a < k; a += blockDim.x) {
    int32_t v = cidx[a];
    int rk = 0;
    for (int q = 0; q < k; ++q) rk += cidx[q] < v;
    Sb[rk] = v;
  }
}

// a2, R28 box mode: bucket b's set = every observation inside the
// bucket box enlarged by beta l_d per axis, ascending index, padded with -1 to k
// (a padded slot is a decoupled far-away dummy in the factor: exact, see k_bucket_factor*).
// Bounds left to right without FMA, as the oracle's.  cnt_max: the largest set.
__global__ void __launch_bounds__(256) k_box_sets(Geom g, const double* __restrict__ X, int64_t m, int k,
                                                  double bl0, double bl1, double bl2, int32_t* __restrict__ S,
                                                  int* __restrict__ cnt_max, int* __restrict__ cnt, int b0) {
  __shared__ int s_base;
  __shared__ int s_wcnt[8];
  const int b = b0 + blockIdx.x;
  const int bi[3] = {b % g.nb[0], (b / g.nb[0]) % g.nb[1], b / (g.nb[0] * g.nb[1])};
  const double bw[3] = {bl0, bl1, bl2};
  double lo[3], hi[3];
  for (int d = 0; d < 3; ++d) {
    lo[d] = __dsub_rn(__dadd_rn(g.lo[d], __dmul_rn((double)(bi[d] * g.bs), g.h[d])), bw[d]);
    hi[d] = __dadd_rn(__dadd_rn(g.lo[d], __dmul_rn((double)((bi[d] + 1) * g.bs), g.h[d])), bw[d]);
  }
  int32_t* Sb = S + (int64_t)b * k;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int64_t i0 = 0; i0 < m; i0 += blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    bool in = i < m;
    for (int d = 0; d < 3 && in; ++d) {
      const double x = X[3 * i + d];
      in = x >= lo[d] && x < hi[d];
    }
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    if (lane == 0) s_wcnt[wid] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      before += w < wid ? s_wcnt[w] : 0;
      total += s_wcnt[w];
    }
    const int slot = s_base + before + __popc(bal & ((1u << lane) - 1u));
    if (in && slot < k) Sb[slot] = (int32_t)i;
    __syncthreads();
    if (threadIdx.x == 0) s_base += total;
    __syncthreads();
  }
  const int n = s_base;
  for (int a = n + threadIdx.x; a < k; a += blockDim.x) Sb[a] = -1;
  if (threadIdx.x == 0) {
    atomicMax(cnt_max, n);
    cnt[b] = n;
  }
}

// R28b (local_mode 2, the |M'| cap): a bucket whose beta-box holds more than k
// observations takes its k-NN set (R2) instead
__global__ void k_box_cap(const int* __restrict__ cnt, int nbuckets, int k, const int32_t* __restrict__ S_knn,
                          int32_t* __restrict__ S, int b0) {
  const int b = b0 + blockIdx.x;
  if (b >= nbuckets || cnt[b] <= k) return;
  for (int a = threadIdx.x; a < k; a += blockDim.x) S[(int64_t)b * k + a] = S_knn[(int64_t)b * k + a];
}

// padded slot a of a box set: a far-away dummy observation, decoupled from everything
// (every kernel value with it is exactly 0, its own variance sigma_f^2 + nugget) with
// value m0, so alpha_a = 0 and its row of L^-1 K is 0: the factor of the real set exactly
__device__ __forceinline__ double dummy_coord(int a, int d) { return 1e20 * (double)(a + 1) * (double)(d + 1); }

// a3: per-bucket factor.  Block layout in bdata: [L^-1 in the DMMA A-fragment
// layout (la_size(k), common.cuh)] [alpha (k)] [x (k)] [y (k)] [z (k)].
// USE_SMEM is a template parameter so that the factor and L^-1 live in pointers the
// compiler knows to be shared (LDS/STS); a runtime choice makes them generic (LD/ST).
template <bool USE_SMEM>
__global__ void __launch_bounds__(FACT_THREADS) k_bucket_factor(KernParams kp, int k, const double* __restrict__ X,
                                                                const double* __restrict__ yobs,
                                                                const int32_t* __restrict__ S,
                                                                double* __restrict__ bdata, int64_t bstride,
                                                                double* __restrict__ gscratch,
                                                                int* __restrict__ derr, int b0) {
  extern __shared__ double sm[];
  __shared__ int s_ok;
  __shared__ double s_piv;
  const int b = b0 + blockIdx.x;
  const int tid = threadIdx.x, bd = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = bd >> 5;
  const int64_t tri = tri_size(k);
  const int64_t LA = la_size(k);
  double* sx = sm;
  double* sy = sx + k;
  double* sz = sy + k;
  double* rr = sz + k;
  double* vv = rr + k;
  double* A;
  double* Li;
  if (USE_SMEM) {
    A = vv + k;
    Li = A + tri;
  } else {
    A = gscratch + (int64_t)b * (tri + (int64_t)k * (k + 1));
    Li = A + tri;
  }
  const int32_t* Sb = S + (int64_t)b * k;
  double* out = bdata + (int64_t)b * bstride;
  for (int a = tid; a < k; a += bd) {
    int64_t o = Sb[a];
    if (o < 0) {   // R28 padding: decoupled far-away dummy (exact, see dummy_coord)
      sx[a] = dummy_coord(a, 0);
      sy[a] = dummy_coord(a, 1);
      sz[a] = dummy_coord(a, 2);
      rr[a] = 0.0;
    } else {
      sx[a] = X[3 * o];
      sy[a] = X[3 * o + 1];
      sz[a] = X[3 * o + 2];
      rr[a] = yobs[o] - kp.m0;
    }
    out[LA + k + a] = sx[a];
    out[LA + 2 * k + a] = sy[a];
    out[LA + 3 * k + a] = sz[a];
  }
  bool ok = false;
  for (int attempt = 0; attempt < 4 && !ok; ++attempt) {
    double jit = attempt == 0 ? 0.0 : 1e-10 * kp.var * (attempt == 1 ? 1.0 : attempt == 2 ? 10.0 : 100.0);
    __syncthreads();
    for (int j = wid; j < k; j += nw) {
      double* colj = A + tri_col(j, k) - j;
      for (int i = j + lane; i < k; i += 32) {
        double r2 = kern_r2(kp, sx[i] - sx[j], sy[i] - sy[j], sz[i] - sz[j]);
        colj[i] = kern_from_r2(kp, r2) + (i == j ? kp.nugget + jit : 0.0);
      }
    }
    if (tid == 0) s_ok = 1;
    // right-looking Cholesky, column by column
    for (int j = 0; j < k; ++j) {
      __syncthreads();
      double* colj = A + tri_col(j, k) - j;
      if (tid == 0) {
        double d = colj[j];
        if (!(d > 0.0)) {
          s_ok = 0;
        } else {
          d = sqrt(d);
          colj[j] = d;
          s_piv = d;
        }
      }
      __syncthreads();
      if (!s_ok) break;
      double piv = s_piv;
      for (int i = j + 1 + tid; i < k; i += bd) colj[i] = colj[i] / piv;
      __syncthreads();
      // trailing update, 4 columns per warp pass (colj[i] shared, 4 independent
      // load-FMA-store chains per lane)
      for (int l0 = j + 1 + 4 * wid; l0 < k; l0 += 4 * nw) {
        double lj[4];
        double* cl[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int l = min(l0 + c, k - 1);
          lj[c] = colj[l];
          cl[c] = A + tri_col(l, k) - l;
        }
        for (int i = l0 + lane; i < k; i += 32) {
          const double ci = colj[i];
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (l0 + c <= i) cl[c][i] = fma(-ci, lj[c], cl[c][i]);
        }
      }
    }
    __syncthreads();
    ok = s_ok != 0;
  }
  if (!ok) {
    if (tid == 0) atomicOr(derr, DERR_FACTOR);
    return;
  }
  // L^-1 = X by a right-looking sweep on a dense row-major X (row stride k + 1):
  // X starts as I; at step p row p is final once divided by L_pp, then every
  // later row subtracts L_ip X[p][:] (warp per row, lanes over columns j <= p)
  const int ldx = k + 1;
  for (int64_t e = tid; e < (int64_t)k * ldx; e += bd) Li[e] = 0.0;
  __syncthreads();
  for (int j = tid; j < k; j += bd) Li[(int64_t)j * ldx + j] = 1.0;
  for (int p = 0; p < k; ++p) {
    __syncthreads();
    const double lpp = A[tri_col(p, k)];
    double* xp = Li + (int64_t)p * ldx;
    for (int j = tid; j <= p; j += bd) xp[j] = xp[j] / lpp;
    __syncthreads();
    const double* colp = A + tri_col(p, k) - p;
    // 4 rows per warp pass (xp[j] shared, 4 independent chains per lane)
    for (int i0 = p + 1 + 4 * wid; i0 < k; i0 += 4 * nw) {
      double li[4];
      double* xr[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = min(i0 + r, k - 1);
        li[r] = colp[i];
        xr[r] = Li + (int64_t)i * ldx;
      }
      for (int j = lane; j <= p; j += 32) {
        const double xpj = xp[j];
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (i0 + r < k) xr[r][j] = fma(-li[r], xpj, xr[r][j]);
      }
    }
  }
  __syncthreads();
  // alpha = L^-T (L^-1 r)
  for (int i = tid; i < k; i += bd) {
    const double* xi = Li + (int64_t)i * ldx;
    double s = 0.0;
    for (int j = 0; j <= i; ++j) s = fma(xi[j], rr[j], s);
    vv[i] = s;
  }
  __syncthreads();
  for (int j = tid; j < k; j += bd) {
    double s = 0.0;
    for (int i = j; i < k; ++i) s = fma(Li[(int64_t)i * ldx + j], vv[i], s);
    out[LA + j] = s;
  }
  for (int64_t e = tid; e < LA; e += bd) {
    const int64_t blk = e >> 5;
    const int ln = (int)(e & 31);
    int rt = (int)((sqrt(4.0 * (double)blk + 1.0) - 1.0) * 0.5);
    while ((int64_t)(rt + 1) * (rt + 2) <= blk) ++rt;
    while ((int64_t)rt * (rt + 1) > blk) --rt;
    const int js = (int)(blk - (int64_t)rt * (rt + 1));
    const int i = 8 * rt + (ln >> 2), j = 4 * js + (ln & 3);
    out[e] = (i < k && j <= i) ? Li[(int64_t)i * ldx + j] : 0.0;
  }
}

// a3, blocked (k <= 128): the same factor with 8x8 blocks on the FP64 tensor cores.
// Dense row-major K_y in smem (row stride KP + 4 = 4 mod 8 doubles: the DMMA
// fragment loads are bank-conflict free), padding rows/columns = identity.
//   Cholesky, right-looking, panel J: (1) warp 0 factors the 8x8 diagonal block
//   (lane r owns row r; shuffles) and its inverse T_J; (2) panel A_IJ <- A_IJ T_J^T;
//   (3) trailing A_{I1,I2} -= A_{I1,J} A_{I2,J}^T -- 2 DMMA.8x8x4 per block.
//   L^-1 = X in place, block row I: S_J = sum_{K=J}^{I-1} L_IK X_KJ (DMMA), then
//   X_IJ = -T_I S_J, X_II = T_I.
// 3 + 2 barriers per block (vs 5 per column unblocked).  Same jitter retry (R15).
constexpr int FB = 8;                  // block size

// 1 / sqrt(x), x > 0: MUFU.RSQ64H seed and two Newton steps (~1 ulp); NaN for x <= 0
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-0.5 * x, y * y, 1.5);
  y = y * fma(-0.5 * x, y * y, 1.5);
  return x > 0.0 ? y : __longlong_as_double(0x7ff8000000000000ll);
}
__device__ __forceinline__ void dmma_f(double a, double b, double& d0, double& d1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// GMEM: K_y / X live in a per-CTA global scratch (L2-resident) instead of shared
// memory (k > 128); CTAs loop over buckets.
template <bool GMEM, int MINB>
__global__ void __launch_bounds__(FACT_THREADS, MINB) k_bucket_factor_blk(KernParams kp, int k, int nbk,
                                                                    const double* __restrict__ X,
                                                                    const double* __restrict__ yobs,
                                                                    const int32_t* __restrict__ S,
                                                                    double* __restrict__ bdata, int64_t bstride,
                                                                    double* __restrict__ gscratch,
                                                                    int* __restrict__ derr, int b0) {
  extern __shared__ double sm[];
  __shared__ int s_ok;
  const int tid = threadIdx.x, bd = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = bd >> 5;
  const int KP = (k + FB - 1) & ~(FB - 1), nb = KP / FB, ST = KP + 4;
  const int64_t LA = la_size(k);
  double* sx = sm;
  double* sy = sx + KP;
  double* sz = sy + KP;
  double* rr = sz + KP;
  double* vv = rr + KP;
  double* sT = vv + KP;                  // nb blocks of 8 x 12 (stride 12: conflict-free)
  double* Srow = sT + nb * FB * 12;      // nb blocks of 8 x 12: S_J of the inverse's block row
  double* A = GMEM ? gscratch + (int64_t)blockIdx.x * KP * ST : Srow + nb * FB * 12;   // KP x ST
  const int lr = lane >> 2, lc = lane & 3;
  for (int b = b0 + blockIdx.x; b < nbk; b += gridDim.x) {   // buckets [b0, nbk)
  __syncthreads();
  const int32_t* Sb = S + (int64_t)b * k;
  double* out = bdata + (int64_t)b * bstride;
  for (int a = tid; a < k; a += bd) {
    int64_t o = Sb[a];
    if (o < 0) {   // R28 padding: decoupled far-away dummy (exact, see dummy_coord)
      sx[a] = dummy_coord(a, 0);
      sy[a] = dummy_coord(a, 1);
      sz[a] = dummy_coord(a, 2);
      rr[a] = 0.0;
    } else {
      sx[a] = X[3 * o];
      sy[a] = X[3 * o + 1];
      sz[a] = X[3 * o + 2];
      rr[a] = yobs[o] - kp.m0;
    }
    out[LA + k + a] = sx[a];
    out[LA + 2 * k + a] = sy[a];
    out[LA + 3 * k + a] = sz[a];
  }
  auto Ab = [&](int I, int J) { return A + (int64_t)(FB * I) * ST + FB * J; };   // block (I, J)
  bool ok = false;
  for (int attempt = 0; attempt < 4 && !ok; ++attempt) {
    const double jit = attempt == 0 ? 0.0 : 1e-10 * kp.var * (attempt == 1 ? 1.0 : attempt == 2 ? 10.0 : 100.0);
    __syncthreads();
    // lower triangle of K_y (+ identity padding rows), warp per row, lanes over columns
    for (int i = wid; i < KP; i += nw) {
      double* Ai = A + (int64_t)i * ST;
      if (i < k) {
        const double xi = sx[i], yi = sy[i], zi = sz[i];
        for (int j = lane; j <= i; j += 32) {
          const double r2 = kern_r2(kp, xi - sx[j], yi - sy[j], zi - sz[j]);
          Ai[j] = kern_from_r2(kp, r2) + (i == j ? kp.nugget + jit : 0.0);
        }
      } else {
        for (int j = lane; j <= i; j += 32) Ai[j] = i == j ? 1.0 : 0.0;
      }
    }
    if (tid == 0) s_ok = 1;
    __syncthreads();
    for (int J = 0; J < nb; ++J) {
      // (1) diagonal block: Cholesky + inverse by warp 0, lane r < 8 owns row r
      if (wid == 0) {
        double d[FB];
        double* D = Ab(J, J);
#pragma unroll
        for (int c = 0; c < FB; ++c) d[c] = (lane < FB && c <= lane) ? D[lane * ST + c] : 0.0;
        bool bad = false;
        double rp[FB];   // 1 / pivot (every lane): the panel solve below multiplies
#pragma unroll
        for (int j = 0; j < FB; ++j) {
          const double pj = __shfl_sync(0xffffffffu, d[j], j);
          if (!(pj > 0.0)) bad = true;
          const double rinv = rsqrt_nr(pj);
          rp[j] = rinv;
          const double piv = pj * rinv;
          if (lane == j) d[j] = piv;
          else if (lane > j && lane < FB) d[j] = d[j] * rinv;
#pragma unroll
          for (int c = j + 1; c < FB; ++c) {
            const double lcj = __shfl_sync(0xffffffffu, d[j], c);
            if (lane >= c && lane < FB) d[c] = fma(-d[j], lcj, d[c]);
          }
        }
        if (lane < FB) {
#pragma unroll
          for (int c = 0; c < FB; ++c)
            if (c <= lane) D[lane * ST + c] = d[c];
        }
        // T = L_JJ^-1, lane c < 8 solves column c: L t = e_c (rows p = c..7)
        __syncwarp();
        if (lane < FB) {
          double t[FB];
#pragma unroll
          for (int p = 0; p < FB; ++p) {
            double sacc = (p == lane) ? 1.0 : 0.0;
#pragma unroll
            for (int q = 0; q < p; ++q) sacc = fma(-D[p * ST + q], t[q], sacc);
            t[p] = p < lane ? 0.0 : sacc * rp[p];
          }
          double* T = sT + J * FB * 12;
#pragma unroll
          for (int p = 0; p < FB; ++p) T[p * 12 + lane] = t[p];
        }
        if (bad && lane == 0) s_ok = 0;
      }
      __syncthreads();
      if (!s_ok) break;
      // (2) panel: A_IJ <- A_IJ T_J^T  (D[r][c] = sum_t A_IJ[r][t] T[c][t])
      const double* T = sT + J * FB * 12;
      for (int I = J + 1 + wid; I < nb; I += nw) {
        double* P = Ab(I, J);
        const double a0 = P[lr * ST + lc], a1 = P[lr * ST + 4 + lc];
        const double b0 = T[lr * 12 + lc], b1 = T[lr * 12 + 4 + lc];
        double d0 = 0.0, d1 = 0.0;
        dmma_f(a0, b0, d0, d1);
        dmma_f(a1, b1, d0, d1);
        __syncwarp();
        P[lr * ST + 2 * lc] = d0;
        P[lr * ST + 2 * lc + 1] = d1;
      }
      __syncthreads();
      // (3) trailing: A_{I1,I2} -= A_{I1,J} A_{I2,J}^T for J < I2 <= I1
      {
        const int m = nb - J - 1, npair = m * (m + 1) / 2;
        for (int idx = wid; idx < npair; idx += nw) {   // pair idx = i1 (i1 + 1) / 2 + i2, i2 <= i1
            int i1 = (int)((sqrtf(8.0f * (float)idx + 1.0f) - 1.0f) * 0.5f);
            while ((i1 + 1) * (i1 + 2) / 2 <= idx) ++i1;
            while (i1 * (i1 + 1) / 2 > idx) --i1;
            const int i2 = idx - i1 * (i1 + 1) / 2;
            const int I1 = J + 1 + i1, I2 = J + 1 + i2;
            const double* P1 = Ab(I1, J);
            const double* P2 = Ab(I2, J);
            double* C = Ab(I1, I2);
            double d0 = C[lr * ST + 2 * lc], d1 = C[lr * ST + 2 * lc + 1];
            dmma_f(-P1[lr * ST + lc], P2[lr * ST + lc], d0, d1);
            dmma_f(-P1[lr * ST + 4 + lc], P2[lr * ST + 4 + lc], d0, d1);
            C[lr * ST + 2 * lc] = d0;
            C[lr * ST + 2 * lc + 1] = d1;
          }
      }
      __syncthreads();
    }
    __syncthreads();
    ok = s_ok != 0;
  }
  if (!ok) {
    if (tid == 0) atomicOr(derr, DERR_FACTOR);
    continue;
  }
  // L^-1 in place, block row by block row
  for (int I = 0; I < nb; ++I) {
    // S_J = sum_{K=J}^{I-1} L_IK X_KJ for J < I (warp w: J = w, w + nw, ...)
    for (int J = wid; J < I; J += nw) {
      double d0 = 0.0, d1 = 0.0;
      for (int K = J; K < I; ++K) {
        const double* Lb = Ab(I, K);
        const double* Xb = Ab(K, J);
        // B[t][c] = X_KJ[t][c]: lane holds X_KJ[t0 + lc][lr]
        dmma_f(Lb[lr * ST + lc], Xb[lc * ST + lr], d0, d1);
        dmma_f(Lb[lr * ST + 4 + lc], Xb[(4 + lc) * ST + lr], d0, d1);
      }
      double* Sj = Srow + J * FB * 12;
      Sj[lr * 12 + 2 * lc] = d0;
      Sj[lr * 12 + 2 * lc + 1] = d1;
    }
    __syncthreads();   // row I of L is consumed; S_J of this row are in Srow
    const double* T = sT + I * FB * 12;
    for (int J = wid; J < I; J += nw) {
      const double* Sj = Srow + J * FB * 12;
      double d0 = 0.0, d1 = 0.0;
      dmma_f(-T[lr * 12 + lc], Sj[lc * 12 + lr], d0, d1);
      dmma_f(-T[lr * 12 + 4 + lc], Sj[(4 + lc) * 12 + lr], d0, d1);
      double* Bk = Ab(I, J);
      Bk[lr * ST + 2 * lc] = d0;
      Bk[lr * ST + 2 * lc + 1] = d1;
    }
    if (wid == nw - 1) {
      double* Dg = Ab(I, I);
      for (int e = lane; e < FB * FB; e += 32) {   // full block: T's upper triangle is 0
        const int r = e >> 3, c = e & 7;
        Dg[r * ST + c] = T[r * 12 + c];
      }
    }
    __syncthreads();
  }
  // alpha = L^-T (L^-1 r)
  for (int i = tid; i < k; i += bd) {
    const double* xi = A + (int64_t)i * ST;
    double sacc = 0.0;
    for (int j = 0; j <= i; ++j) sacc = fma(xi[j], rr[j], sacc);
    vv[i] = sacc;
  }
  __syncthreads();
  for (int j = tid; j < k; j += bd) {
    double sacc = 0.0;
    for (int i = j; i < k; ++i) sacc = fma(A[(int64_t)i * ST + j], vv[i], sacc);
    out[LA + j] = sacc;
  }
  // L^-1 as DMMA A-fragments: warp per 32-double block (row tile rt, column step js)
  for (int64_t blk = wid; blk < (LA >> 5); blk += nw) {
    int rt = (int)((sqrtf(4.0f * (float)blk + 1.0f) - 1.0f) * 0.5f);
    while ((int64_t)(rt + 1) * (rt + 2) <= blk) ++rt;
    while ((int64_t)rt * (rt + 1) > blk) --rt;
    const int js = (int)(blk - (int64_t)rt * (rt + 1));
    const int i = 8 * rt + (lane >> 2), j = 4 * js + (lane & 3);
    out[blk * 32 + lane] = (i < k && j <= i) ? A[(int64_t)i * ST + j] : 0.0;
  }
  }   // bucket loop
}

size_t bucket_factor_blk_smem(int k, bool gmem) {
  const int KP = (k + FB - 1) & ~(FB - 1), nb = KP / FB;
  return sizeof(double) * (5 * (size_t)KP + 2 * (size_t)nb * FB * 12 + (gmem ? 0 : (size_t)KP * (KP + 4)));
}

// NEXT-2: SGPR bucket factor.  Eq. 1 restricted to the bucket's local
// inducing points S (its k nearest, or its beta-box set, R28):
//   mu(x) = m0 + k_x^T W (mu_S - m0),  Sigma = K - k^T W k + k^T W A_SS W k,
// W = (K_SS + jitter)^-1 = L^-T L^-1.  With v = L^-1 k and B = L^-1 A_SS L^-T the two
// subtracted terms are v^T (I - B) v; I - B (eigenvalues in [0, 1]) is factored as
// U U^T with U upper triangular (Cholesky of the index-reversed P (I - B) P = R R^T,
// U = P R P; PSD clamp as R14), and G = U^T L^-1 is lower triangular with
// Sigma = K - ||G k||^2.  So the bucket block [G as DMMA A-fragments | beta = W (mu_S -
// m0) | x_S] has the same form as the GP-regression block (G = L^-1 there) and every
// downstream kernel is unchanged.  No explicit W: on the ill-conditioned fuzz draws
// (cond(K_SS) ~ 1e10-1e11) this keeps Sigma within ~1e-9 sigma_f^2 of an extended-
// precision evaluation, where the former C = W - W A W factor lost ~1e-6.
// Persistent CTAs with dense k x k global scratch (5 k^2 doubles each).
__global__ void __launch_bounds__(FACT_THREADS) k_bucket_factor_sgpr(KernParams kp, int k, const double* __restrict__ X,
                                                                     const double* __restrict__ muM,
                                                                     const double* __restrict__ AM, int64_t m,
                                                                     const int32_t* __restrict__ S,
                                                                     double* __restrict__ bdata, int64_t bstride,
                                                                     double* __restrict__ scratch, int nbuckets,
                                                                     int* __restrict__ derr, int b0) {
  extern __shared__ double sm[];
  __shared__ int s_ok;
  __shared__ double s_piv;
  const int tid = threadIdx.x, bd = blockDim.x;
  const int64_t kk = (int64_t)k * k;
  double* M0 = scratch + (int64_t)blockIdx.x * 5 * kk;   // K -> L, later P (I - B) P -> R
  double* M1 = M0 + kk;                                  // L^-1
  double* M2 = M1 + kk;                                  // T = L^-1 A_SS, later G
  double* M3 = M2 + kk;                                  // A_SS; M3 + kk: L^-1 r
  double* sx = sm;
  double* sy = sx + k;
  double* sz = sy + k;
  double* rr = sz + k;
  const int64_t LA = la_size(k);
  for (int b = b0 + blockIdx.x; b < nbuckets; b += gridDim.x) {   // buckets [b0, nbuckets)
    const int32_t* Sb = S + (int64_t)b * k;
    double* out = bdata + (int64_t)b * bstride;
    __syncthreads();
    for (int a = tid; a < k; a += bd) {
      int64_t o = Sb[a];
      if (o < 0) {   // R28 padding of a beta-box set: decoupled far-away dummy, no A term
        sx[a] = dummy_coord(a, 0); sy[a] = dummy_coord(a, 1); sz[a] = dummy_coord(a, 2);
        rr[a] = 0.0;
      } else {
        sx[a] = X[3 * o]; sy[a] = X[3 * o + 1]; sz[a] = X[3 * o + 2];
        rr[a] = muM[o] - kp.m0;
      }
      out[LA + k + a] = sx[a]; out[LA + 2 * k + a] = sy[a]; out[LA + 3 * k + a] = sz[a];
    }
    bool ok = false;
    for (int attempt = 0; attempt < 4 && !ok; ++attempt) {
      double jit = kp.nugget + (attempt == 0 ? 0.0 : 1e-10 * kp.var * (attempt == 1 ? 1.0 : attempt == 2 ? 10.0 : 100.0));
      __syncthreads();
      for (int64_t e = tid; e < kk; e += bd) {
        int i = (int)(e / k), j = (int)(e % k);
        double r2 = kern_r2(kp, sx[i] - sx[j], sy[i] - sy[j], sz[i] - sz[j]);
        M0[e] = kern_from_r2(kp, r2) + (i == j ? jit : 0.0);
      }
      if (tid == 0) s_ok = 1;
      for (int j = 0; j < k; ++j) {
        __syncthreads();
        if (tid == 0) {
          double d = M0[(int64_t)j * k + j];
          if (!(d > 0.0)) s_ok = 0;
          else { d = sqrt(d); M0[(int64_t)j * k + j] = d; s_piv = d; }
        }
        __syncthreads();
        if (!s_ok) break;
        const double piv = s_piv;
        for (int i = j + 1 + tid; i < k; i += bd) M0[(int64_t)i * k + j] /= piv;
        __syncthreads();
        for (int64_t e = tid; e < (int64_t)(k - j - 1) * (k - j - 1); e += bd) {
          int i = j + 1 + (int)(e / (k - j - 1)), l = j + 1 + (int)(e % (k - j - 1));
          if (l <= i) M0[(int64_t)i * k + l] -= M0[(int64_t)i * k + j] * M0[(int64_t)l * k + j];
        }
      }
      __syncthreads();
      ok = s_ok != 0;
    }
    if (!ok) {
      if (tid == 0) atomicOr(derr, DERR_FACTOR);
      continue;
    }
    // L^-1 (column forward substitutions)
    for (int j = tid; j < k; j += bd) {
      for (int i = 0; i < j; ++i) M1[(int64_t)i * k + j] = 0.0;
      M1[(int64_t)j * k + j] = 1.0 / M0[(int64_t)j * k + j];
      for (int i = j + 1; i < k; ++i) {
        double s = 0.0;
        for (int p = j; p < i; ++p) s = fma(M0[(int64_t)i * k + p], M1[(int64_t)p * k + j], s);
        M1[(int64_t)i * k + j] = -s / M0[(int64_t)i * k + i];
      }
    }
    // A_SS (padding slots of a box set: 0 -- a decoupled dummy carries no A term)
    for (int64_t e = tid; e < kk; e += bd) {
      const int32_t si = Sb[e / k], sj = Sb[e % k];
      M3[e] = (si >= 0 && sj >= 0) ? AM[(int64_t)si * m + sj] : 0.0;
    }
    __syncthreads();   // L^-1 and A_SS complete
    // beta = W r = L^-T (L^-1 r) (two triangular products: no explicit W)
    double* tv = M3 + kk;
    for (int i = tid; i < k; i += bd) {
      double s = 0.0;
      for (int l = 0; l <= i; ++l) s = fma(M1[(int64_t)i * k + l], rr[l], s);
      tv[i] = s;
    }
    __syncthreads();
    for (int i = tid; i < k; i += bd) {
      double s = 0.0;
      for (int l = i; l < k; ++l) s = fma(M1[(int64_t)l * k + i], tv[l], s);
      out[LA + i] = s;
    }
    // T = L^-1 A_SS (into M2)
    for (int64_t e = tid; e < kk; e += bd) {
      int i = (int)(e / k), j = (int)(e % k);
      double s = 0.0;
      for (int l = 0; l <= i; ++l) s = fma(M1[(int64_t)i * k + l], M3[(int64_t)l * k + j], s);
      M2[e] = s;
    }
    __syncthreads();
    // I - B with B = T L^-T = L^-1 A_SS L^-T, symmetrised, stored index-reversed:
    // M0[i][j] = (I - B)[k-1-i][k-1-j].  Eq. 1's two subtracted terms then combine as
    // K - k^T W k + k^T W A W k = K - v^T (I - B) v with v = L^-1 k: I - B has its
    // eigenvalues in [0, 1] and no explicit W = K_SS^-1 enters (the W - W A W form lost
    // cond(K_SS) eps to cancellation)
    for (int64_t e = tid; e < kk; e += bd) {
      int i = (int)(e / k), j = (int)(e % k);
      double s1 = 0.0, s2 = 0.0;
      for (int l = 0; l <= j; ++l) s1 = fma(M2[(int64_t)i * k + l], M1[(int64_t)j * k + l], s1);
      for (int l = 0; l <= i; ++l) s2 = fma(M2[(int64_t)j * k + l], M1[(int64_t)i * k + l], s2);
      M0[(int64_t)(k - 1 - i) * k + (k - 1 - j)] = (i == j ? 1.0 : 0.0) - 0.5 * (s1 + s2);
    }
    __syncthreads();
    // clamped Cholesky of P (I - B) P = R R^T (in place, lower), tol = 1e-12 max diag;
    // I - B = U U^T with U = P R P upper triangular
    if (tid == 0) {
      double md = 0.0;
      for (int i = 0; i < k; ++i) md = fmax(md, M0[(int64_t)i * k + i]);
      s_piv = 1e-12 * md;
    }
    __syncthreads();
    const double tol = s_piv;
    for (int j = 0; j < k; ++j) {
      __syncthreads();
      if (tid == 0) {
        double d = M0[(int64_t)j * k + j];
        s_ok = d > tol;
        M0[(int64_t)j * k + j] = d > tol ? sqrt(d) : 0.0;
      }
      __syncthreads();
      const bool live = s_ok;
      const double piv = M0[(int64_t)j * k + j];
      for (int i = j + 1 + tid; i < k; i += bd) M0[(int64_t)i * k + j] = live ? M0[(int64_t)i * k + j] / piv : 0.0;
      __syncthreads();
      for (int64_t e = tid; e < (int64_t)(k - j - 1) * (k - j - 1); e += bd) {
        int i = j + 1 + (int)(e / (k - j - 1)), l = j + 1 + (int)(e % (k - j - 1));
        if (l <= i) M0[(int64_t)i * k + l] -= M0[(int64_t)i * k + j] * M0[(int64_t)l * k + j];
      }
    }
    __syncthreads();
    // G = U^T L^-1 (lower): G[i][j] = sum_{p=j..i} U[p][i] L^-1[p][j], U[p][i] = R[k-1-p][k-1-i];
    // Sigma = K - ||G k||^2, the GP-regression form of the block (G = L^-1 there)
    for (int64_t e = tid; e < kk; e += bd) {
      int i = (int)(e / k), j = (int)(e % k);
      double s = 0.0;
      for (int pp = j; pp <= i; ++pp) s = fma(M0[(int64_t)(k - 1 - pp) * k + (k - 1 - i)], M1[(int64_t)pp * k + j], s);
      M2[e] = j <= i ? s : 0.0;
    }
    __syncthreads();
    // G written as DMMA A-fragments
    for (int64_t e = tid; e < LA; e += bd) {
      const int64_t blk = e >> 5;
      const int ln = (int)(e & 31);
      int rt = (int)((sqrt(4.0 * (double)blk + 1.0) - 1.0) * 0.5);
      while ((int64_t)(rt + 1) * (rt + 2) <= blk) ++rt;
      while ((int64_t)rt * (rt + 1) > blk) --rt;
      const int js = (int)(blk - (int64_t)rt * (rt + 1));
      const int i = 8 * rt + (ln >> 2), j = 4 * js + (ln & 3);
      out[e] = (i < k && j <= i) ? M2[(int64_t)i * k + j] : 0.0;
    }
  }
}

// ------------------------------------------------------------------- host
static int ilog2_ceil(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return l;
}

static double host_kern(const KernParams& p, const double* a, const double* b) {
  double r2 = 0.0;
  for (int d = 0; d < 3; ++d) {
    double t = (a[d] - b[d]) * p.inv_ls[d];
    r2 += t * t;
  }
  if (p.kind == LCP_K_SE) return p.var * std::exp(-0.5 * r2);
  double r = std::sqrt(r2), s = SQRT5 * r;
  return p.var * (1.0 + s + (5.0 / 3.0) * r2) * std::exp(-s);
}

lcp_status_t fit_impl(Ctx& c, const double* xyz, const double* yv, int64_t m, int on_device,
                      const lcp_kernel_t* kern, int k, const lcp_grid_t* grid, const lcp_opts_t* opts,
                      const double* AM) {
  NvtxRange nvtx_("lcp_fit");
  if (!xyz || !yv || !kern || !grid) return set_err(c, LCP_EINVAL, "fit: null argument");
  if (m < 1 || k < 1 || (int64_t)k > m) return set_err(c, LCP_EINVAL, "fit: need 1 <= k <= m");
  if (k > 1024 && (int64_t)k != m) return set_err(c, LCP_EINVAL, "fit: k > 1024 requires k == m");
  if (!(kern->variance > 0) || !(kern->nugget >= 0) || !std::isfinite(kern->variance) ||
      !std::isfinite(kern->nugget) || !std::isfinite(kern->prior_mean) ||
      (kern->kind != LCP_K_SE && kern->kind != LCP_K_MATERN52))
    return set_err(c, LCP_EINVAL, "fit: bad kernel parameters");
  for (int d = 0; d < 3; ++d)
    if (!(kern->lengthscale[d] > 0) || !std::isfinite(kern->lengthscale[d]) || grid->cells[d] < 1 ||
        !(grid->hi[d] > grid->lo[d]) || !std::isfinite(grid->lo[d]) || !std::isfinite(grid->hi[d]) ||
        grid->cells[d] > (1 << 20))
      return set_err(c, LCP_EINVAL, "fit: bad lengthscale or grid");
  lcp_opts_t o{};
  o.bucket_log2 = 0;
  o.h_full = 2;
  o.precision = LCP_FP64;
  o.slab_rank = 0;
  o.slab_count = 1;
  o.slab_level = 0;
  o.keep_records = 0;
  o.extreme_iters = 0;
  if (opts) o = *opts;
  if (o.local_mode < 0 || o.local_mode > 2) return set_err(c, LCP_EINVAL, "fit: bad local_mode");
  if (o.local_mode >= 1 && !(o.beta > 0.0 && std::isfinite(o.beta))) return set_err(c, LCP_EINVAL, "fit: beta must be > 0");
  if (o.precision != LCP_FP64 && o.precision != LCP_FP32) return set_err(c, LCP_EINVAL, "fit: bad precision");
  if (o.precision == LCP_FP32 && k > 128) return set_err(c, LCP_EINVAL, "fit: the FP32 posterior needs k <= 128");
  if (o.extreme_iters < 0 || o.extreme_iters > 1000) return set_err(c, LCP_EINVAL, "fit: extreme_iters not in [0, 1000]");
  if (o.slab_count < 1) o.slab_count = 1;
  int cmax = std::max(grid->cells[0], std::max(grid->cells[1], grid->cells[2]));
  int lfull = ilog2_ceil(cmax);
  if (o.bucket_log2 < 0 || o.bucket_log2 > lfull || o.h_full < 0 || o.slab_rank < 0 ||
      o.slab_rank >= o.slab_count)
    return set_err(c, LCP_EINVAL, "fit: bad options (bucket_log2 / h_full / slab)");
  // candidate lattice of a node: (2^min(h, h_full) + 1)^3 vertices, indexed in 32 bits
  if (std::min(o.h_full, lfull) > 10)
    return set_err(c, LCP_EINVAL, "fit: h_full > 10 (lattice of > 2^30 vertices per node)");
  if (o.slab_count > 1 && o.slab_level > lfull)
    return set_err(c, LCP_EINVAL, "fit: slab_level must be <= Lfull (or <= 0: automatic)");

  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, c.stream);

  c.fitted = false;
  c.vcache_valid = false;
  c.slab_planned = false;
  c.kern = *kern;
  c.grid = *grid;
  c.opts = o;
  c.m = m;
  c.k = k;
  KernParams& kp = c.kp;
  kp.kind = kern->kind;
  kp.var = kern->variance;
  for (int d = 0; d < 3; ++d) kp.inv_ls[d] = 1.0 / kern->lengthscale[d];
  kp.nugget = kern->nugget;
  kp.m0 = kern->prior_mean;
  Geom& g = c.g;
  g.lfull = lfull;
  g.bs_log2 = lfull - o.bucket_log2;
  g.bs = 1 << g.bs_log2;
  g.h_full = o.h_full;
  for (int d = 0; d < 3; ++d) {
    g.lo[d] = grid->lo[d];
    g.cells[d] = grid->cells[d];
    g.h[d] = (grid->hi[d] - grid->lo[d]) / (double)grid->cells[d];
    g.sB[d] = (double)g.bs * g.h[d];
    g.nb[d] = (grid->cells[d] + g.bs - 1) / g.bs;
  }
  g.nbuckets = g.nb[0] * g.nb[1] * g.nb[2];
  // prior covariance among the 8 corners (depends on h only)
  for (int cc = 0; cc < 8; ++cc)
    for (int dd = 0; dd <= cc; ++dd) {
      double a[3] = {(cc & 1) * g.h[0], ((cc >> 1) & 1) * g.h[1], (cc >> 2) * g.h[2]};
      double b[3] = {(dd & 1) * g.h[0], ((dd >> 1) & 1) * g.h[1], (dd >> 2) * g.h[2]};
      c.kcc[cc * (cc + 1) / 2 + dd] = host_kern(kp, a, b);
    }
  int64_t tri = tri_size(k);
  c.bstride = (la_size(k) + 4 * (int64_t)k + 1) & ~1ll;
  const int nbk = g.nbuckets;

  cudaError_t e;
#define CK(x)                                  \
  do {                                         \
    e = (x);                                   \
    if (e != cudaSuccess) return cuda_err(c, e, #x); \
  } while (0)
  CK(c.X.ensure(sizeof(double) * 3 * m));
  CK(c.y.ensure(sizeof(double) * m));
  CK(c.obs_bucket.ensure(sizeof(int32_t) * m));
  CK(c.obs_key.ensure(sizeof(uint64_t) * m));
  CK(c.obs_sorted_key.ensure(sizeof(uint64_t) * m));
  CK(c.obs_sorted_idx.ensure(sizeof(int32_t) * m));
  CK(c.obs_by_bucket.ensure(sizeof(int64_t) * m));
  CK(c.bcount.ensure(sizeof(int64_t) * nbk));
  CK(c.bstart.ensure(sizeof(int64_t) * nbk));
  // sharded fit (opts.fit_shard with slab_count > 1): this rank computes the k-NN sets and
  // factors of buckets [b0, b1) only -- an equal split of the bucket index range padded to
  // nbp = slab_count x per buckets -- and the caller all-gathers the blocks in place
  // (lcp_fit_shard_buffers) before lcp_fit_finish
  const bool shard = o.fit_shard != 0 && o.slab_count > 1;
  const int per = shard ? (nbk + o.slab_count - 1) / o.slab_count : nbk;
  const int nbp = shard ? per * o.slab_count : nbk;
  const int b0 = shard ? std::min(nbk, o.slab_rank * per) : 0;
  const int b1 = shard ? std::min(nbk, b0 + per) : nbk;
  c.shard_per = per;
  c.fit_pending = false;
  CK(c.S.ensure(sizeof(int32_t) * (size_t)nbp * k));
  CK(c.bdata.ensure(sizeof(double) * (size_t)nbp * c.bstride));
  CK(c.obs_mu.ensure(sizeof(double) * m));
  CK(c.obs_sd.ensure(sizeof(double) * m));
  CK(c.derr.ensure(sizeof(int) * 4));
  CK(c.knn_fail.ensure(sizeof(int) * (nbk + 1)));
  CK(c.cell_bucket.ensure(sizeof(int32_t) * m));
  CK(cudaMemsetAsync(c.derr.p, 0, sizeof(int) * 4, c.stream));
  if (on_device) {
    CK(cudaMemcpyAsync(c.X.p, xyz, sizeof(double) * 3 * m, cudaMemcpyDeviceToDevice, c.stream));
    CK(cudaMemcpyAsync(c.y.p, yv, sizeof(double) * m, cudaMemcpyDeviceToDevice, c.stream));
  } else {
    CK(cudaMemcpyAsync(c.X.p, xyz, sizeof(double) * 3 * m, cudaMemcpyHostToDevice, c.stream));
    CK(cudaMemcpyAsync(c.y.p, yv, sizeof(double) * m, cudaMemcpyHostToDevice, c.stream));
  }
  const double* X = c.X.as<double>();
  unsigned gm = (unsigned)((m + 255) / 256);
  // a1
  k_obs_bin<<<gm, 256, 0, c.stream>>>(g, X, c.y.as<double>(), m, c.obs_bucket.as<int32_t>(), c.obs_key.as<uint64_t>(),
                                      c.derr.as<int>());
  ++c.n_launch;
  CK(group_by_bucket(c, c.obs_bucket.as<int32_t>(), m, c.obs_by_bucket.as<int64_t>()));
  k_bucket_ranges<<<(nbk + 255) / 256, 256, 0, c.stream>>>(c.gcount.as<int64_t>(), c.goff.as<int64_t>(), nbk,
                                                          c.bcount.as<int64_t>(), c.bstart.as<int64_t>());
  ++c.n_launch;
  k_obs_rank<<<gm, 256, 0, c.stream>>>(c.obs_key.as<uint64_t>(), m, c.obs_sorted_key.as<uint64_t>(),
                                      c.obs_sorted_idx.as<int32_t>());
  ++c.n_launch;
  CK(cudaGetLastError());
  // occupancy bitmaps for the three finest octree levels (the preliminary test of a node
  // without observations then skips its two binary searches); up to 2^30 cells
  c.occ_heights = g.lfull <= 10 ? std::min(3, g.lfull + 1) : 0;
  for (int h = 0; h < c.occ_heights; ++h) {
    const size_t words = ((((size_t)1) << (3 * (g.lfull - h))) + 31) / 32;
    CK(c.occ[h].ensure(sizeof(uint32_t) * words));
    CK(cudaMemsetAsync(c.occ[h].p, 0, sizeof(uint32_t) * words, c.stream));
  }
  if (c.occ_heights > 0) {
    k_occ_set<<<gm, 256, 0, c.stream>>>(c.obs_key.as<uint64_t>(), m, c.occ_heights, c.occ[0].as<uint32_t>(),
                                        c.occ[1].as<uint32_t>(), c.occ[2].as<uint32_t>());
    ++c.n_launch;
    CK(cudaGetLastError());
  }
  // a2
  auto knn_sets = [&](int32_t* Sout) -> cudaError_t {
    int r0 = 0;
    double dens = (double)m / nbk;
    while (r0 < 64 && std::pow(2.0 * r0 + 1.0, 3) * dens < (double)k) ++r0;
    size_t smem = sizeof(double) * KNN_CMAX + sizeof(int32_t) * KNN_CMAX + sizeof(int32_t) * (k + 2) +
                  sizeof(double) * (k + 1);
    cudaError_t ee;
    if ((ee = cudaFuncSetAttribute(k_knn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
      return ee;
    if ((ee = cudaFuncSetAttribute(k_knn_brute, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
        cudaSuccess)
      return ee;
    int* nfail_dev = c.knn_fail.as<int>();
    int* list_dev = nfail_dev + 1;
    if ((ee = cudaMemsetAsync(nfail_dev, 0, sizeof(int), c.stream)) != cudaSuccess) return ee;
    if (b1 <= b0) return cudaSuccess;
    k_knn<<<b1 - b0, KNN_THREADS, smem, c.stream>>>(kp, g, X, m, k, c.bstart.as<int64_t>(), c.bcount.as<int64_t>(),
                                                  c.obs_by_bucket.as<int64_t>(), Sout, list_dev, nfail_dev, r0, b0);
    ++c.n_launch;
    if ((ee = cudaGetLastError()) != cudaSuccess) return ee;
    int nfail = 0;
    if ((ee = cudaMemcpyAsync(&nfail, nfail_dev, sizeof(int), cudaMemcpyDeviceToHost, c.stream)) != cudaSuccess)
      return ee;
    if ((ee = cudaStreamSynchronize(c.stream)) != cudaSuccess) return ee;
    c.knn_fallbacks = nfail;
    if (nfail > 0) {
      k_knn_brute<<<nfail, KNN_THREADS, smem, c.stream>>>(kp, g, X, m, k, list_dev, Sout);
      ++c.n_launch;
      if ((ee = cudaGetLastError()) != cudaSuccess) return ee;
    }
    return cudaSuccess;
  };
  c.n_capped = 0;
  if (o.local_mode >= 1) {
    int32_t* S_knn = nullptr;
    if (o.local_mode == 2) {   // the |M'| cap: k-NN sets for the buckets whose box overflows
      CK(c.S_knn.ensure(sizeof(int32_t) * (size_t)nbk * k));
      S_knn = c.S_knn.as<int32_t>();
      CK(knn_sets(S_knn));
    }
    CK(c.box_cnt.ensure(sizeof(int) * (size_t)nbk));
    int* cmax = c.knn_fail.as<int>();
    CK(cudaMemsetAsync(cmax, 0, sizeof(int), c.stream));
    if (b1 > b0) {
      k_box_sets<<<b1 - b0, 256, 0, c.stream>>>(g, X, m, k, o.beta * kern->lengthscale[0],
                                                o.beta * kern->lengthscale[1], o.beta * kern->lengthscale[2],
                                                c.S.as<int32_t>(), cmax, c.box_cnt.as<int>(), b0);
      ++c.n_launch;
    }
    CK(cudaGetLastError());
    int hmax = 0;
    CK(cudaMemcpyAsync(&hmax, cmax, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    if (o.local_mode == 1) c.knn_fallbacks = 0;
    c.max_set = std::min(hmax, k);
    if (hmax > k && o.local_mode == 1)
      return set_err(c, LCP_EINVAL, "fit: a beta-box holds " + std::to_string(hmax) + " observations > k = " +
                                        std::to_string(k) + " (raise k, lower beta, or use local_mode 2)");
    if (hmax > k && b1 > b0) {
      k_box_cap<<<b1 - b0, 128, 0, c.stream>>>(c.box_cnt.as<int>(), nbk, k, S_knn, c.S.as<int32_t>(), b0);
      ++c.n_launch;
      CK(cudaGetLastError());
      std::vector<int> hc(b1 - b0);
      CK(cudaMemcpyAsync(hc.data(), c.box_cnt.as<int>() + b0, sizeof(int) * (size_t)(b1 - b0),
                         cudaMemcpyDeviceToHost, c.stream));
      CK(cudaStreamSynchronize(c.stream));
      for (int v : hc) c.n_capped += v > k;
    }
  } else {
    CK(knn_sets(c.S.as<int32_t>()));
  }
  // a3
  if (AM) {
    // NEXT-2 SGPR factors (A_M uploaded as m x m)
    CK(c.sgpr_A.ensure(sizeof(double) * (size_t)m * m));
    CK(cudaMemcpyAsync(c.sgpr_A.p, AM, sizeof(double) * (size_t)m * m,
                       on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
    k_check_finite<<<std::min<int64_t>(((int64_t)m * m + 255) / 256, 4 * (int64_t)c.sm_count * 8), 256, 0,
                     c.stream>>>(c.sgpr_A.as<double>(), (int64_t)m * m, c.derr.as<int>());
    ++c.n_launch;
    int grid_f = std::max(1, std::min(b1 - b0, c.sm_count * 2));
    CK(c.fscratch.ensure(sizeof(double) * 5 * (size_t)k * k * grid_f));
    size_t smem = sizeof(double) * 4 * (size_t)k;
    if (b1 > b0) {
      k_bucket_factor_sgpr<<<grid_f, FACT_THREADS, smem, c.stream>>>(kp, k, X, c.y.as<double>(),
                                                                     c.sgpr_A.as<double>(), m, c.S.as<int32_t>(),
                                                                     c.bdata.as<double>(), c.bstride,
                                                                     c.fscratch.as<double>(), b1, c.derr.as<int>(), b0);
      ++c.n_launch;
    }
    CK(cudaGetLastError());
  } else {
    size_t head = sizeof(double) * 5 * (size_t)k;
    size_t full = head + sizeof(double) * ((size_t)tri + (size_t)k * (k + 1));
    int use_smem = full <= 220 * 1024;
    size_t smem = use_smem ? full : head;
    double* gs = nullptr;
    if (!use_smem) {
      CK(c.fscratch.ensure(sizeof(double) * ((size_t)tri + (size_t)k * (k + 1)) * nbk));
      gs = c.fscratch.as<double>();
    }
    static const bool blk_off = [] {
      const char* v = std::getenv("LCP_FACTOR_BLOCKED");
      return v && v[0] == '0';
    }();
    // The blocked factor keeps its k x k working matrix in a per-CTA L2-resident global
    // scratch (GMEM) with 4 CTAs (64 registers each) per SM: the factorisation is barrier-
    // and latency-bound, and 4 concurrent buckets per SM beat 1 with the matrix in shared
    // memory (c5 fit 23.3 -> 19.5 ms).  LCP_FACTOR_SMEM=1 selects the shared-memory variant
    // when the matrix fits (k <= 128).
    static const bool smem_variant = [] {
      const char* v = std::getenv("LCP_FACTOR_SMEM");
      return v && v[0] == '1';
    }();
    if (!blk_off && bucket_factor_blk_smem(k, true) <= 220 * 1024) {
      const bool gm = !(smem_variant && bucket_factor_blk_smem(k, false) <= 220 * 1024);
      const size_t sb = bucket_factor_blk_smem(k, gm);
      const int KPf = (k + FB - 1) & ~(FB - 1);
      const int nfb = b1 - b0;
      unsigned gridf = (unsigned)std::max(1, nfb);
      double* gsf = nullptr;
      if (nfb <= 0) {
      } else if (gm) {
        // many buckets (k <= 256): 4 CTAs of <= 64 registers per SM; otherwise 2 unconstrained
        const bool four = KPf <= 256 && nfb >= 2 * (int64_t)c.sm_count;
        gridf = (unsigned)std::min<int64_t>(nfb, (four ? 4 : 2) * (int64_t)c.sm_count);
        CK(c.fscratch.ensure(sizeof(double) * (size_t)gridf * KPf * (KPf + 4)));
        gsf = c.fscratch.as<double>();
        auto kf = four ? k_bucket_factor_blk<true, 4> : k_bucket_factor_blk<true, 1>;
        CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
        kf<<<gridf, FACT_THREADS, sb, c.stream>>>(kp, k, b1, X, c.y.as<double>(), c.S.as<int32_t>(),
                                                  c.bdata.as<double>(), c.bstride, gsf, c.derr.as<int>(), b0);
        ++c.n_launch;
      } else {
        CK(cudaFuncSetAttribute(k_bucket_factor_blk<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
        k_bucket_factor_blk<false, 1><<<gridf, FACT_THREADS, sb, c.stream>>>(kp, k, b1, X, c.y.as<double>(),
                                                                             c.S.as<int32_t>(), c.bdata.as<double>(),
                                                                             c.bstride, nullptr, c.derr.as<int>(), b0);
        ++c.n_launch;
      }
    } else if (b1 <= b0) {
    } else if (use_smem) {
      CK(cudaFuncSetAttribute(k_bucket_factor<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_bucket_factor<true><<<b1 - b0, FACT_THREADS, smem, c.stream>>>(kp, k, X, c.y.as<double>(), c.S.as<int32_t>(),
                                                                       c.bdata.as<double>(), c.bstride, gs,
                                                                       c.derr.as<int>(), b0);
      ++c.n_launch;
    } else {
      CK(cudaFuncSetAttribute(k_bucket_factor<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_bucket_factor<false><<<b1 - b0, FACT_THREADS, smem, c.stream>>>(kp, k, X, c.y.as<double>(), c.S.as<int32_t>(),
                                                                        c.bdata.as<double>(), c.bstride, gs,
                                                                        c.derr.as<int>(), b0);
      ++c.n_launch;
    }
    CK(cudaGetLastError());
  }
  cudaEventRecord(e1, c.stream);
  CK(cudaStreamSynchronize(c.stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  c.t.fit_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
#undef CK
  if (shard) {   // the caller exchanges the bucket blocks, then lcp_fit_finish runs a4
    lcp_status_t st = check_device_errors(c);
    if (st != LCP_OK) return st;
    c.fit_pending = true;
    return LCP_OK;
  }
  return fit_finish_impl(c);
}

// a4 (observation marginals, every bucket factor present) and the context state after a fit
lcp_status_t fit_finish_impl(Ctx& c) {
  NvtxRange nvtx_("lcp_fit_finish");
  cudaError_t e;
#define CK(x)                                  \
  do {                                         \
    e = (x);                                   \
    if (e != cudaSuccess) return cuda_err(c, e, #x); \
  } while (0)
  const Geom& g = c.g;
  const int64_t m = c.m;
  const double* X = c.X.as<double>();
  const unsigned gm = (unsigned)((m + 255) / 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, c.stream);
  // a4: observation marginals (grouped by bucket)
  k_gather_i32<<<gm, 256, 0, c.stream>>>(c.obs_bucket.as<int32_t>(), c.obs_by_bucket.as<int64_t>(), m,
                                         c.cell_bucket.as<int32_t>());
  ++c.n_launch;
  CK(launch_marginals(c, Q_OBS, c.obs_by_bucket.as<int64_t>(), c.cell_bucket.as<int32_t>(), m, X,
                      c.obs_mu.as<double>(), c.obs_sd.as<double>(), 0, nullptr));
  cudaEventRecord(e1, c.stream);
  CK(cudaStreamSynchronize(c.stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  c.t.fit_ms += ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  c.fit_pending = false;
  lcp_status_t st = check_device_errors(c);
  if (st != LCP_OK) return st;
  // the vertex cache covers every grid vertex
  int64_t nv = (int64_t)(g.cells[0] + 1) * (g.cells[1] + 1) * (g.cells[2] + 1);
  c.n_vertices = nv;
  CK(c.vcache.ensure(sizeof(double2) * nv));
  CK(c.vstate.ensure(sizeof(uint32_t) * ((nv + 31) / 32)));
  CK(cudaMemsetAsync(c.vstate.p, 0, sizeof(uint32_t) * ((nv + 31) / 32), c.stream));
  c.vcache_valid = true;
  c.fitted = true;
#undef CK
  return fused_setup(c);
}

}  // namespace lcp
