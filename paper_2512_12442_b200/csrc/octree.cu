// octree.cu -- lcp_octree_refine: SURVEY §8(a) rows a5-a6.
//
// Alg. 1 run level-synchronously: the frontier of level L
// is a Morton-ordered array of node keys; every node is evaluated by one warp:
//   k_node_prelim : M~ = observations in the node (a contiguous range of the
//                   Morton-sorted observations), p1 = max P(Y_i < th),
//                   p2 = max P(Y_i > th) (lines 3-5), the case
//                   (R8, R9) and, unless case 1, requests for the candidate
//                   lattice vertices (R6) whose marginals are not cached yet;
//   k_marginals   : local-GP marginals of the requested vertices (marginals.cu);
//   k_node_bound  : B_l, B_u over the lattice and U = 1 - B_l^d - B_u^d in log
//                   space (Eq. 3-4; R7, R9);
//   k_node_counts / exclusive scan / k_emit : stream compaction of the refined
//                   nodes into the next frontier (8 children in Morton order,
//                   lines 14-21) or, at max depth, into the leaf-cell list (line 13).
#include <algorithm>
#include <cmath>

#include "ctx.h"

namespace lcp {

struct Lattice {
  int64_t base[3], vmax[3], stride;
  int cnt[3];
};

__device__ __forceinline__ Lattice node_lattice(const Geom& g, int h, int i, int j, int k) {
  Lattice L;
  int a[3] = {i, j, k};
  int st = h - g.h_full > 0 ? h - g.h_full : 0;
  L.stride = (int64_t)1 << st;
  for (int d = 0; d < 3; ++d) {
    L.base[d] = (int64_t)a[d] << h;
    int64_t e = L.base[d] + ((int64_t)1 << h);
    L.vmax[d] = e < g.cells[d] ? e : g.cells[d];
    L.cnt[d] = (int)((L.vmax[d] - L.base[d] + L.stride - 1) / L.stride) + 1;
  }
  return L;
}

// q < cnt0 cnt1 cnt2 <= (2^h_full + 1)^3: 32-bit division (the 64-bit one is a ~70-instruction
// routine, and the finest levels decode 8 corners for each of up to 1.3e8 nodes)
__device__ __forceinline__ int64_t lattice_vertex(const Geom& g, const Lattice& L, int64_t q64) {
  const unsigned q = (unsigned)q64, c0 = (unsigned)L.cnt[0], c1 = (unsigned)L.cnt[1];
  const unsigned r = q / c0;
  const int t0 = (int)(q - r * c0);
  const unsigned r2 = r / c1;
  const int t1 = (int)(r - r2 * c1);
  const int t2 = (int)r2;
  int64_t v0 = t0 < L.cnt[0] - 1 ? L.base[0] + t0 * L.stride : L.vmax[0];
  int64_t v1 = t1 < L.cnt[1] - 1 ? L.base[1] + t1 * L.stride : L.vmax[1];
  int64_t v2 = t2 < L.cnt[2] - 1 ? L.base[2] + t2 * L.stride : L.vmax[2];
  return vertex_id(g, v0, v1, v2);
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t n, uint64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// a4 per isovalue: tails of the observation marginals, Morton order
__global__ void k_obs_probs(const int32_t* __restrict__ sidx, const double* __restrict__ mu,
                            const double* __restrict__ sd, int64_t m, double theta, double* __restrict__ plo,
                            double* __restrict__ phi) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  int o = sidx[r];
  double s2 = sd[o] * SQRT2;
  plo[r] = 0.5 * erfc((mu[o] - theta) / s2);
  phi[r] = 0.5 * erfc((theta - mu[o]) / s2);
}

// G lanes per node (G | 32): 1 at the finest level, up to a warp at coarse ones.
template <int G>
__device__ __forceinline__ double group_max(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int G>
__device__ __forceinline__ double group_min(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int G>
__global__ void k_node_prelim(Geom g, int level, const uint64_t* __restrict__ front, int64_t nF,
                              const uint64_t* __restrict__ skey, const double* __restrict__ plo,
                              const double* __restrict__ phi, int64_t m, double alpha,
                              int8_t* __restrict__ ncase, int8_t* __restrict__ nref, double* __restrict__ np1,
                              double* __restrict__ np2, double* __restrict__ nU, uint32_t* __restrict__ vmask,
                              int64_t* __restrict__ req, unsigned long long* __restrict__ nreq,
                              const uint32_t* __restrict__ occ, int lattice_all) {
  int64_t n = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int sub = threadIdx.x % G;
  const bool live = n < nF;
  int i = 0, j = 0, k = 0;
  if (live) node_unkey(front[n], i, j, k);
  const int h = g.lfull - level;
  int64_t a = 0, b = 0;
  if (live && sub == 0) {
    uint64_t mk = morton3(i, j, k);
    if (!occ || ((occ[mk >> 5] >> (mk & 31)) & 1u)) {   // bitmap: no observation in the node -> empty
      a = lower_bound_u64(skey, m, mk << (3 * h));
      b = lower_bound_u64(skey, m, (mk + 1) << (3 * h));
    }
  }
  if (G > 1) {
    a = __shfl_sync(0xffffffffu, a, 0, G);
    b = __shfl_sync(0xffffffffu, b, 0, G);
  }
  double p1 = -1.0, p2 = -1.0;
  for (int64_t r = a + sub; r < b; r += G) {
    p1 = fmax(p1, plo[r]);
    p2 = fmax(p2, phi[r]);
  }
  p1 = group_max<G>(p1);
  p2 = group_max<G>(p2);
  const bool any = b > a;
  const int cs = !any ? 0 : ((p1 > alpha && p2 > alpha) ? 1 : (p2 <= alpha ? 2 : 3));
  if (live && sub == 0) {
    ncase[n] = (int8_t)cs;
    np1[n] = p1;
    np2[n] = p2;
    if (cs == 1) {
      nref[n] = 1;
      nU[n] = 1.0;
    }
  }
  if (!live || (cs == 1 && !lattice_all)) return;   // lattice_all: the slab weights read it
  Lattice L = node_lattice(g, h, i, j, k);
  int64_t nc = (int64_t)L.cnt[0] * L.cnt[1] * L.cnt[2];
  for (int64_t q = sub; q < nc; q += G) {
    int64_t v = lattice_vertex(g, L, q);
    uint32_t bit = 1u << (v & 31);
    if (vmask[v >> 5] & bit) continue;
    uint32_t old = atomicOr(&vmask[v >> 5], bit);
    if (!(old & bit)) req[atomicAdd(nreq, 1ull)] = v;
  }
}

__global__ void k_req_bucket(Geom g, const int64_t* __restrict__ req, int64_t n, int32_t* __restrict__ bkt) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) bkt[q] = vertex_bucket(g, req[q]);
}

__global__ void k_gather_req(const int64_t* __restrict__ req, const int32_t* __restrict__ bkt,
                             const int64_t* __restrict__ perm, int64_t n, int64_t* __restrict__ req_s,
                             int32_t* __restrict__ bkt_s) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  int64_t p = perm[q];
  req_s[q] = req[p];
  bkt_s[q] = bkt[p];
}

// U of Eq. 4 in log space from the extreme z values (R9):
// Q_lo = max P(Y > th) = erfc(-zmax)/2, Q_hi = max P(Y < th) = erfc(zmin)/2
__device__ __forceinline__ double bound_U(int cs, double d, double zmax, double zmin) {
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
  return U;
}

__device__ __forceinline__ double node_dcount(const Lattice& L) {
  return (double)(L.vmax[0] - L.base[0] + 1) * (double)(L.vmax[1] - L.base[1] + 1) *
         (double)(L.vmax[2] - L.base[2] + 1);
}

// vcache[v] = (mu_v, 1 / (sigma_v sqrt 2)).  If ext != nullptr the lattice
// extremes and their vertices (first lattice index on ties, like the oracle's
// x-fastest scan) are kept for the continuous search (NEXT-1).
template <int G>
__global__ void k_node_bound(Geom g, int level, const uint64_t* __restrict__ front, int64_t nF, double theta,
                             double alpha, const int8_t* __restrict__ ncase, const double2* __restrict__ vcache,
                             int8_t* __restrict__ nref, double* __restrict__ nU, double* __restrict__ ext_z,
                             int64_t* __restrict__ ext_v) {
  int64_t n = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int sub = threadIdx.x % G;
  const bool live = n < nF && ncase[n] != 1;
  const int cs = live ? ncase[n] : 1;
  int i = 0, j = 0, k = 0;
  if (live) node_unkey(front[n], i, j, k);
  const int h = g.lfull - level;
  Lattice L = node_lattice(g, h, i, j, k);
  int64_t nc = live ? (int64_t)L.cnt[0] * L.cnt[1] * L.cnt[2] : 0;
  double zmax = -INFINITY, zmin = INFINITY;
  int64_t qmax = INT64_MAX, qmin = INT64_MAX;
  for (int64_t q = sub; q < nc; q += G) {
    double2 ms = vcache[lattice_vertex(g, L, q)];
    double z = (ms.x - theta) * ms.y;
    if (z > zmax) { zmax = z; qmax = q; }
    if (z < zmin) { zmin = z; qmin = q; }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    double zx = __shfl_xor_sync(0xffffffffu, zmax, o), zn = __shfl_xor_sync(0xffffffffu, zmin, o);
    int64_t qx = __shfl_xor_sync(0xffffffffu, qmax, o), qn = __shfl_xor_sync(0xffffffffu, qmin, o);
    if (zx > zmax || (zx == zmax && qx < qmax)) { zmax = zx; qmax = qx; }
    if (zn < zmin || (zn == zmin && qn < qmin)) { zmin = zn; qmin = qn; }
  }
  if (!live || sub != 0) return;
  double U = bound_U(cs, node_dcount(L), zmax, zmin);
  nU[n] = U;
  nref[n] = U > alpha ? 1 : 0;
  if (ext_z) {
    ext_z[2 * n] = zmax;
    ext_z[2 * n + 1] = zmin;
    ext_v[2 * n] = lattice_vertex(g, L, qmax);
    ext_v[2 * n + 1] = lattice_vertex(g, L, qmin);
  }
}

// NEXT-1 (R26): continuous refinement of the lattice extremes (extreme.cu)
cudaError_t launch_node_extreme(Ctx& c, int level, const uint64_t* front, int64_t nF, double theta,
                                double alpha, const int8_t* ncase, int8_t* nref, double* nU, const double* ext_z,
                                const int64_t* ext_v);

__global__ void k_node_records(int level, const uint64_t* __restrict__ front, int64_t nF,
                               const int8_t* __restrict__ ncase, const int8_t* __restrict__ nref,
                               const double* __restrict__ np1, const double* __restrict__ np2,
                               const double* __restrict__ nU, lcp_node_rec_t* __restrict__ out,
                               unsigned long long* __restrict__ stats) {
  __shared__ unsigned int s_cnt[5];
  if (threadIdx.x < 5) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool live = n < nF;
  int cs = live ? ncase[n] : -1;
  bool rf = live && nref[n];
  if (live && out) {
    lcp_node_rec_t r;
    node_unkey(front[n], r.i, r.j, r.k);
    r.level = level;
    r.ncase = cs;
    r.refine = rf;
    r.p1 = np1[n];
    r.p2 = np2[n];
    r.U = nU[n];
    out[n] = r;
  }
  // per-level statistics: warp ballots, one shared atomic per warp, one global per block
  unsigned bq[5];
#pragma unroll
  for (int q = 0; q < 4; ++q) bq[q] = __ballot_sync(0xffffffffu, cs == q);
  bq[4] = __ballot_sync(0xffffffffu, rf);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int q = 0; q < 5; ++q)
      if (bq[q]) atomicAdd(&s_cnt[q], __popc(bq[q]));
  }
  __syncthreads();
  if (threadIdx.x < 5 && s_cnt[threadIdx.x]) atomicAdd(&stats[threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
}

// NEXT-4 level field: the cells of a node that stops
// at this level (pruned, or refined at max depth) get the level.  G lanes per node.
template <int G>
__global__ void k_fill_level(Geom g, int level, int max_depth, const uint64_t* __restrict__ front, int64_t nF,
                             const int8_t* __restrict__ nref, uint8_t* __restrict__ field) {
  int64_t n = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int sub = threadIdx.x % G;
  if (n >= nF) return;
  if (nref[n] && level < max_depth) return;   // continues below
  int i, j, k;
  node_unkey(front[n], i, j, k);
  const int h = g.lfull - level;
  const int64_t side = (int64_t)1 << h;
  const int64_t b0 = (int64_t)i * side, b1 = (int64_t)j * side, b2 = (int64_t)k * side;
  const int64_t e0 = min(b0 + side, (int64_t)g.cells[0]) - b0, e1 = min(b1 + side, (int64_t)g.cells[1]) - b1,
                e2 = min(b2 + side, (int64_t)g.cells[2]) - b2;
  const int64_t tot = e0 * e1 * e2;
  for (int64_t t = sub; t < tot; t += G) {
    const int64_t x = b0 + t % e0, y = b1 + (t / e0) % e1, z = b2 + t / (e0 * e1);
    field[x + (int64_t)g.cells[0] * (y + (int64_t)g.cells[1] * z)] = (uint8_t)level;
  }
}

// Slab weights (identical on every rank): per z-layer of the slab level, the expected
// leaf work of its refined nodes -- 1 + 1024 x (fraction of the node's lattice vertices
// whose marginal is uncertain, |z| < zs, i.e. both tails > alpha / 8) x (clipped cells /
// full node cells).  Thin-shell fields (NEXT-4) put their leaves near few layers.
__global__ void k_layer_weight(Geom g, int level, const uint64_t* __restrict__ front, int64_t nF,
                               const int8_t* __restrict__ nref, const double2* __restrict__ vcache, double theta,
                               double zs, int nz, unsigned long long* __restrict__ hist) {
  int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= nF || !nref[n]) return;
  int i, j, k;
  node_unkey(front[n], i, j, k);
  if (k >= nz) return;
  const int h = g.lfull - level;
  Lattice L = node_lattice(g, h, i, j, k);
  const int64_t nc = (int64_t)L.cnt[0] * L.cnt[1] * L.cnt[2];
  int64_t unc = 0;
  for (int64_t q = 0; q < nc; ++q) {
    const double2 ms = vcache[lattice_vertex(g, L, q)];
    unc += fabs((ms.x - theta) * ms.y) < zs;
  }
  const uint64_t cells = (uint64_t)(L.vmax[0] - L.base[0]) * (L.vmax[1] - L.base[1]) * (L.vmax[2] - L.base[2]);
  const uint64_t full = 1ull << (3 * h);
  const uint64_t w = 1 + (uint64_t)((1024.0 * (double)unc / (double)nc) * ((double)cells / (double)full));
  atomicAdd(&hist[k], (unsigned long long)w);
}

// Slab filter of a rank: the children of refined level-slab_level nodes
// are kept iff the node's z index is in [z0, z1); leaf cells emitted at a level <=
// slab_level are kept iff their z is in [cz0, cz1).  slab_level < 0: whole domain.
struct Slab {
  int level, z0, z1;
  int64_t cz0, cz1;
};

// children / leaf counts of refined nodes
__global__ void k_node_counts(Geom g, int level, int max_depth, const uint64_t* __restrict__ front, int64_t nF,
                              const int8_t* __restrict__ nref, Slab sl, int64_t* __restrict__ cnt) {
  int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= nF) return;
  if (!nref[n]) {
    cnt[n] = 0;
    return;
  }
  int i, j, k;
  node_unkey(front[n], i, j, k);
  int h = g.lfull - level;
  if (level < max_depth) {
    if (level == sl.level && (k < sl.z0 || k >= sl.z1)) {
      cnt[n] = 0;
      return;
    }
    int64_t cs = (int64_t)1 << (h - 1);
    int c = 0;
    for (int ch = 0; ch < 8; ++ch) {
      int64_t ci = 2 * (int64_t)i + (ch & 1), cj = 2 * (int64_t)j + ((ch >> 1) & 1), ck = 2 * (int64_t)k + (ch >> 2);
      c += ci * cs < g.cells[0] && cj * cs < g.cells[1] && ck * cs < g.cells[2];
    }
    cnt[n] = c;
  } else {
    int64_t side = (int64_t)1 << h;
    int64_t e[3], b[3];
    int a[3] = {i, j, k};
    for (int d = 0; d < 3; ++d) {
      b[d] = (int64_t)a[d] * side;
      e[d] = min(b[d] + side, (int64_t)g.cells[d]);
    }
    if (level <= sl.level) {
      b[2] = max(b[2], sl.cz0);
      e[2] = min(e[2], sl.cz1);
    }
    cnt[n] = e[2] > b[2] ? (e[0] - b[0]) * (e[1] - b[1]) * (e[2] - b[2]) : 0;
  }
}

__global__ void k_emit(Geom g, int level, int max_depth, const uint64_t* __restrict__ front, int64_t nF,
                       const int8_t* __restrict__ nref, const int64_t* __restrict__ offs, Slab sl,
                       uint64_t* __restrict__ next, int64_t* __restrict__ leaves) {
  int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= nF || !nref[n]) return;
  int i, j, k;
  node_unkey(front[n], i, j, k);
  int h = g.lfull - level;
  int64_t o = offs[n];
  if (level < max_depth) {
    if (level == sl.level && (k < sl.z0 || k >= sl.z1)) return;
    int64_t cs = (int64_t)1 << (h - 1);
    for (int ch = 0; ch < 8; ++ch) {
      int64_t ci = 2 * (int64_t)i + (ch & 1), cj = 2 * (int64_t)j + ((ch >> 1) & 1), ck = 2 * (int64_t)k + (ch >> 2);
      bool in = ci * cs < g.cells[0] && cj * cs < g.cells[1] && ck * cs < g.cells[2];
      if (in) next[o++] = node_key(ci, cj, ck);
    }
  } else {
    int64_t side = (int64_t)1 << h;
    int64_t b0 = (int64_t)i * side, b1 = (int64_t)j * side, b2 = (int64_t)k * side;
    int64_t e0 = min(b0 + side, (int64_t)g.cells[0]), e1 = min(b1 + side, (int64_t)g.cells[1]),
            e2 = min(b2 + side, (int64_t)g.cells[2]);
    if (level <= sl.level) {
      b2 = max(b2, sl.cz0);
      e2 = min(e2, sl.cz1);
    }
    for (int64_t z = b2; z < e2; ++z)
      for (int64_t y = b1; y < e1; ++y)
        for (int64_t x = b0; x < e0; ++x) leaves[o++] = x + (int64_t)g.cells[0] * (y + (int64_t)g.cells[1] * z);
  }
}

// The leaf cells of the nodes of a leaf level above the cells (max_depth < Lfull, h >= 2):
// CTAs take (node, chunk of EMIT_CHUNK cells) items grid-stride and write the node's
// clipped cell box in the (z, y, x) order of k_emit's serial loop -- a thread per node
// would write up to 8^h cells alone (max_depth 0 on c4: 8.4 M cells in one thread, 70 ms).
constexpr int64_t EMIT_CHUNK = 4096;
__global__ void k_emit_cells(Geom g, int level, const uint64_t* __restrict__ front, int64_t nF,
                             const int8_t* __restrict__ nref, const int64_t* __restrict__ offs, Slab sl,
                             int64_t nchunk, int64_t* __restrict__ leaves) {
  const int64_t side = (int64_t)1 << (g.lfull - level);
  for (int64_t it = blockIdx.x; it < nF * nchunk; it += gridDim.x) {
    const int64_t n = it / nchunk, c0 = (it % nchunk) * EMIT_CHUNK;
    if (!nref[n]) continue;
    int i, j, k;
    node_unkey(front[n], i, j, k);
    const int64_t b0 = (int64_t)i * side, b1 = (int64_t)j * side;
    int64_t b2 = (int64_t)k * side;
    const int64_t e0 = min(b0 + side, (int64_t)g.cells[0]), e1 = min(b1 + side, (int64_t)g.cells[1]);
    int64_t e2 = min(b2 + side, (int64_t)g.cells[2]);
    if (level <= sl.level) {
      b2 = max(b2, sl.cz0);
      e2 = min(e2, sl.cz1);
    }
    const int64_t ex = e0 - b0, ey = e1 - b1, tot = e2 > b2 ? ex * ey * (e2 - b2) : 0;
    const int64_t c1 = min(tot, c0 + EMIT_CHUNK);
    int64_t* out = leaves + offs[n];
    for (int64_t t = c0 + threadIdx.x; t < c1; t += blockDim.x) {
      const int64_t x = b0 + t % ex, y = b1 + (t / ex) % ey, z = b2 + t / (ex * ey);
      out[t] = x + (int64_t)g.cells[0] * (y + (int64_t)g.cells[1] * z);
    }
  }
}

// z-layers of level L over the grid
int slab_layers_at(const Geom& g, int L) {
  const int64_t side = (int64_t)1 << (g.lfull - L);
  return (int)((g.cells[2] + side - 1) / side);
}

// Automatic slab level: the shallowest level with >= 2 slab_count z-layers (weighted cuts
// need a few layers per rank), at most Lfull - 3 (the brick pass starts below the slab
// level) and at most max_depth.
int auto_slab_level(const Geom& g, int count, int max_depth) {
  const int cap = std::max(1, std::min(max_depth, g.lfull - 3));
  for (int L = 1; L < cap; ++L)
    if (slab_layers_at(g, L) >= 2 * count) return L;
  return cap;
}

// Contiguous z-layer ranges of `count` ranks minimising the largest rank weight (then the
// sum of squared rank weights; ties to the earlier cut), every rank >= 1 layer when there
// are at least `count` layers; equal layer counts when every weight is 0.  Exact dynamic
// programme over (ranks, layers), O(count nz^2) with nz <= 2^10; integer arithmetic only,
// so every rank computes the same cuts.
std::vector<int> slab_cuts(const std::vector<int64_t>& w, int count) {
  const int nz = (int)w.size();
  std::vector<int> cut(count + 1, 0);
  cut[count] = nz;
  std::vector<int64_t> P(nz + 1, 0);
  for (int z = 0; z < nz; ++z) P[z + 1] = P[z] + w[z];
  if (P[nz] == 0) {
    for (int r = 1; r < count; ++r) cut[r] = (int)((int64_t)r * nz / count);
    return cut;
  }
  const bool one_each = nz >= count;
  const int64_t INF = INT64_MAX;
  typedef std::pair<int64_t, double> Cost;   // (max rank weight, sum of squares)
  std::vector<std::vector<Cost>> f(count + 1, std::vector<Cost>(nz + 1, Cost(INF, 0.0)));
  std::vector<std::vector<int>> arg(count + 1, std::vector<int>(nz + 1, 0));
  f[0][0] = Cost(0, 0.0);
  for (int r = 1; r <= count; ++r)
    for (int z = 0; z <= nz; ++z)
      for (int zp = 0; zp <= z; ++zp) {
        if (one_each && zp == z) continue;
        if (f[r - 1][zp].first == INF) continue;
        const int64_t load = P[z] - P[zp];
        const Cost cst(std::max(f[r - 1][zp].first, load), f[r - 1][zp].second + (double)load * (double)load);
        if (cst < f[r][z]) {
          f[r][z] = cst;
          arg[r][z] = zp;
        }
      }
  for (int r = count, z = nz; r > 0; --r) {
    cut[r] = z;
    z = arg[r][z];
  }
  cut[0] = 0;
  return cut;
}

lcp_status_t refine_impl(Ctx& c, double theta, double alpha, int max_depth) {
  NvtxRange nvtx_("lcp_octree_refine");
  if (!c.fitted) return set_err(c, LCP_ESTATE, "refine before fit");
  if (!(alpha > 0.0 && alpha < 0.5)) return set_err(c, LCP_EINVAL, "refine: threshold must be in (0, 0.5)");
  if (max_depth < 0 || max_depth > c.g.lfull) return set_err(c, LCP_EINVAL, "refine: max_depth not in [0, Lfull]");
  if (!std::isfinite(theta)) return set_err(c, LCP_EINVAL, "refine: isovalue not finite");
  const Geom& g = c.g;
  cudaError_t e;
#define CK(x)                                        \
  do {                                               \
    e = (x);                                         \
    if (e != cudaSuccess) return cuda_err(c, e, #x); \
  } while (0)
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, c.stream);
  const int64_t m = c.m;
  CK(c.plo.ensure(sizeof(double) * m));
  CK(c.phi.ensure(sizeof(double) * m));
  CK(c.counters.ensure(sizeof(unsigned long long) * 16));
  if (!c.h_counters) CK(cudaMallocHost(&c.h_counters, sizeof(int64_t) * 16));
  k_obs_probs<<<(unsigned)((m + 255) / 256), 256, 0, c.stream>>>(c.obs_sorted_idx.as<int32_t>(), c.obs_mu.as<double>(),
                                                                 c.obs_sd.as<double>(), m, theta, c.plo.as<double>(),
                                                                 c.phi.as<double>());
  ++c.n_launch;
  CK(c.front[0].ensure(sizeof(uint64_t)));
  uint64_t root = node_key(0, 0, 0);
  CK(cudaMemcpyAsync(c.front[0].p, &root, sizeof(uint64_t), cudaMemcpyHostToDevice, c.stream));
  int cur = 0;
  int64_t nF = 1;
  c.n_leaves = 0;
  c.n_recs = 0;
  c.t.brick_ms = 0;
  c.last_requests = 0;
  c.level_nodes.clear();
  c.level_refined.clear();
  for (int q = 0; q < 4; ++q) c.level_case[q].clear();
  // z-slab of this rank: levels 0..slab_level are evaluated over the whole
  // domain; the cut is placed at slab_level by the first refine after the fit
  Slab sl{-1, 0, 1 << 30, 0, INT64_MAX};
  bool plan_now = false;
  if (c.opts.slab_count > 1) {
    if (c.slab_planned) {
      sl.level = c.slab_L;
    } else {
      const int want = c.opts.slab_level > 0 ? std::min(c.opts.slab_level, g.lfull)
                                             : auto_slab_level(g, c.opts.slab_count, g.lfull);
      sl.level = std::min(want, max_depth);
      plan_now = true;
      c.slab_L = sl.level;
      c.slab_nz = slab_layers_at(g, sl.level);
      if (c.fused && sl.level > g.lfull - 3) c.fused = false;   // bricks must lie below the slab level
    }
    if (!plan_now) {
      sl.z0 = c.slab_z0;
      sl.z1 = c.slab_z1;
      const int64_t side = (int64_t)1 << (g.lfull - c.slab_L);
      sl.cz0 = std::min<int64_t>((int64_t)sl.z0 * side, g.cells[2]);
      sl.cz1 = std::min<int64_t>((int64_t)sl.z1 * side, g.cells[2]);
    }
  }
  unsigned long long* dcnt = c.counters.as<unsigned long long>();
  if (c.level_field)
    CK(cudaMemsetAsync(c.level_field, 0xFF, (size_t)g.cells[0] * g.cells[1] * g.cells[2], c.stream));
  bool early_bricks = false;
  for (int level = 0; level <= max_depth && nF > 0; ++level) {
    NvtxRange nvtx_l("octree level %d", level);
    int h = g.lfull - level;
    CK(c.ncase.ensure(nF));
    CK(c.nref.ensure(nF));
    CK(c.np1.ensure(sizeof(double) * nF));
    CK(c.np2.ensure(sizeof(double) * nF));
    CK(c.nU.ensure(sizeof(double) * nF));
    CK(c.cnt.ensure(sizeof(int64_t) * nF));
    CK(c.offs.ensure(sizeof(int64_t) * nF));
    CK(cudaMemsetAsync(c.nref.p, 0, nF, c.stream));
    int hf = std::min(h, g.h_full);
    int64_t per = ((int64_t)1 << hf) + 1;
    int64_t cap = std::min(nF * per * per * per, c.n_vertices);
    CK(c.req.ensure(sizeof(int64_t) * cap));
    CK(c.req_sorted.ensure(sizeof(int64_t) * cap));
    CK(c.cell_bucket.ensure(sizeof(int32_t) * 2 * cap));
    CK(c.perm.ensure(sizeof(int64_t) * cap));
    CK(cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long) * 16, c.stream));
    const uint64_t* F = c.front[cur].as<uint64_t>();
    // refine-time brick pass over level-(Lfull-2) node keys (aligned 4^3-cell bricks):
    // one pass computes their vertex marginals (the bound's lattice, R6, R10) and the MC
    // records of all their cells (a7-a8), reused by every later leaf pass.  Bricks done
    // earlier in this fit are skipped inside the kernel.
    auto brick_pass = [&](const uint64_t* keys, int64_t nk) -> cudaError_t {
      NvtxRange nvtx_b("brick pass");
      cudaEvent_t b0, b1;
      cudaEventCreate(&b0);
      cudaEventCreate(&b1);
      cudaEventRecord(b0, c.stream);
      const int64_t ch = std::min<int64_t>(nk, BRICK_PASS_CHUNK);
      cudaError_t be = c.post.ensure(sizeof(double) * 44 * 64 * ch);
      for (int64_t off = 0; off < nk && be == cudaSuccess; off += ch) {
        const int64_t nb = std::min(ch, nk - off);
        be = launch_brick_pass(c, keys + off, nb, c.post.as<double>());
        if (be == cudaSuccess) be = launch_chol8_rec(c, keys + off, nb, c.post.as<double>());
      }
      cudaEventRecord(b1, c.stream);
      if (be == cudaSuccess) be = cudaEventSynchronize(b1);
      float bms = 0;
      cudaEventElapsedTime(&bms, b0, b1);
      c.t.brick_ms += bms;
      cudaEventDestroy(b0);
      cudaEventDestroy(b1);
      return be;
    };
    // early pass over the frontier's descendant bricks at level Lfull-4 (64 per node) or
    // Lfull-3 (8 per node), when the previous level refined nearly everything (then nearly
    // every descendant brick would be reached anyway): its vertex marginals serve the
    // spacing-4 / spacing-2 bound lattices of those levels, which otherwise need separate
    // k_marginals passes over 1/64 + 1/8 of all vertices
    static const bool early_env = [] {
      const char* v = std::getenv("LCP_EARLY_BRICK");
      return !(v && v[0] == '0');
    }();
    const int gen = h == 4 ? 2 : (h == 3 ? 1 : 0);
    if (c.fused && c.rec_ready && gen > 0 && !early_bricks && early_env && level >= 1 && level > sl.level &&
        !c.level_nodes.empty() &&
        c.level_refined.back() * 20 >= c.level_nodes.back() * (gen == 2 ? 19 : 18)) {
      const int64_t nk = nF << (3 * gen);
      CK(c.child_bricks.ensure(sizeof(uint64_t) * nk));
      CK(launch_child_bricks(c, F, nF, gen, c.child_bricks.as<uint64_t>()));
      CK(brick_pass(c.child_bricks.as<uint64_t>(), nk));
      early_bricks = true;   // covers every brick of the later frontiers
    }
    if (c.fused && c.rec_ready && h == 2 && !early_bricks) CK(brick_pass(F, nF));
    const int G = h == 0 ? 1 : (h == 1 ? 4 : (h == 2 ? 8 : 32));
    unsigned gw = (unsigned)((nF * G + 255) / 256);
#define PRELIM(GG)                                                                                              \
  k_node_prelim<GG><<<gw, 256, 0, c.stream>>>(g, level, F, nF, c.obs_sorted_key.as<uint64_t>(), c.plo.as<double>(), \
                                               c.phi.as<double>(), m, alpha, c.ncase.as<int8_t>(),                \
                                               c.nref.as<int8_t>(), c.np1.as<double>(), c.np2.as<double>(),       \
                                               c.nU.as<double>(), c.vstate.as<uint32_t>(), c.req.as<int64_t>(), dcnt, \
                                               h < c.occ_heights ? c.occ[h].as<uint32_t>() : nullptr, \
                                               (plan_now && level == sl.level) ? 1 : 0)
    if (G == 1) PRELIM(1);
    else if (G == 4) PRELIM(4);
    else if (G == 8) PRELIM(8);
    else PRELIM(32);
#undef PRELIM
    ++c.n_launch;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(c.h_counters, dcnt, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    int64_t nreq = c.h_counters[0];
    c.last_requests += nreq;
    if (nreq > 0) {
      int32_t* bkt = c.cell_bucket.as<int32_t>();
      int32_t* bkt_s = bkt + cap;
      unsigned gr = (unsigned)((nreq + 255) / 256);
      k_req_bucket<<<gr, 256, 0, c.stream>>>(g, c.req.as<int64_t>(), nreq, bkt);
      ++c.n_launch;
      CK(group_by_bucket(c, bkt, nreq, c.perm.as<int64_t>()));
      k_gather_req<<<gr, 256, 0, c.stream>>>(c.req.as<int64_t>(), bkt, c.perm.as<int64_t>(), nreq,
                                             c.req_sorted.as<int64_t>(), bkt_s);
      ++c.n_launch;
      CK(launch_marginals(c, Q_VERTEX, c.req_sorted.as<int64_t>(), bkt_s, nreq, nullptr, nullptr, nullptr, 0,
                          nullptr));
    }
    const bool ext = c.opts.extreme_iters > 0 && h > g.h_full;   // NEXT-1
    if (ext) {
      CK(c.ext_z.ensure(sizeof(double) * 2 * nF));
      CK(c.ext_v.ensure(sizeof(int64_t) * 2 * nF));
    }
    double* ez = ext ? c.ext_z.as<double>() : nullptr;
    int64_t* ev = ext ? c.ext_v.as<int64_t>() : nullptr;
#define BOUND(GG)                                                                                            \
  k_node_bound<GG><<<gw, 256, 0, c.stream>>>(g, level, F, nF, theta, alpha, c.ncase.as<int8_t>(),             \
                                              c.vcache.as<double2>(), c.nref.as<int8_t>(), c.nU.as<double>(),  \
                                              ez, ev)
    if (G == 1) BOUND(1);
    else if (G == 4) BOUND(4);
    else if (G == 8) BOUND(8);
    else BOUND(32);
#undef BOUND
    ++c.n_launch;
    if (ext) CK(launch_node_extreme(c, level, F, nF, theta, alpha, c.ncase.as<int8_t>(), c.nref.as<int8_t>(),
                                    c.nU.as<double>(), ez, ev));
    lcp_node_rec_t* rec_out = nullptr;
    const bool keep = level < c.opts.keep_records;
    if (keep) {
      CK(c.recs.ensure_keep(sizeof(lcp_node_rec_t) * (c.n_recs + nF), sizeof(lcp_node_rec_t) * c.n_recs, c.stream));
      rec_out = c.recs.as<lcp_node_rec_t>() + c.n_recs;
    }
    unsigned gt = (unsigned)((nF + 255) / 256);
    k_node_records<<<gt, 256, 0, c.stream>>>(level, F, nF, c.ncase.as<int8_t>(), c.nref.as<int8_t>(),
                                             c.np1.as<double>(), c.np2.as<double>(), c.nU.as<double>(), rec_out,
                                             dcnt + 8);
    ++c.n_launch;
    if (c.level_field) {
      if (h <= 2) {
        k_fill_level<1><<<gt, 256, 0, c.stream>>>(g, level, max_depth, F, nF, c.nref.as<int8_t>(), c.level_field);
      } else {
        k_fill_level<32><<<(unsigned)((nF * 32 + 255) / 256), 256, 0, c.stream>>>(g, level, max_depth, F, nF,
                                                                                 c.nref.as<int8_t>(),
                                                                                 c.level_field);
      }
      ++c.n_launch;
    }
    if (plan_now && level == sl.level) {
      // slab weights: refined nodes of this level per z-layer -> contiguous cuts (host)
      const int nz = c.slab_nz;
      CK(c.scan_tmp.ensure(sizeof(unsigned long long) * nz));
      unsigned long long* hist = c.scan_tmp.as<unsigned long long>();
      CK(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * nz, c.stream));
      // zs: 0.5 erfc(zs) = alpha / 8 (bisection; the single-cell survival band of Eq. 4 with d = 8)
      double za = 0.0, zb = 40.0;
      for (int it = 0; it < 200; ++it) {
        const double zm = 0.5 * (za + zb);
        (0.5 * std::erfc(zm) > alpha / 8.0 ? za : zb) = zm;
      }
      k_layer_weight<<<gt, 256, 0, c.stream>>>(g, level, F, nF, c.nref.as<int8_t>(), c.vcache.as<double2>(), theta,
                                               za, nz, hist);
      ++c.n_launch;
      c.slab_w.assign(nz, 0);
      CK(cudaMemcpyAsync(c.slab_w.data(), hist, sizeof(int64_t) * nz, cudaMemcpyDeviceToHost, c.stream));
      CK(cudaStreamSynchronize(c.stream));
      c.slab_cuts = slab_cuts(c.slab_w, c.opts.slab_count);
      c.slab_z0 = c.slab_cuts[c.opts.slab_rank];
      c.slab_z1 = c.slab_cuts[c.opts.slab_rank + 1];
      sl.z0 = c.slab_z0;
      sl.z1 = c.slab_z1;
      const int64_t side = (int64_t)1 << (g.lfull - sl.level);
      sl.cz0 = std::min<int64_t>((int64_t)sl.z0 * side, g.cells[2]);
      sl.cz1 = std::min<int64_t>((int64_t)sl.z1 * side, g.cells[2]);
      // a plan capped by max_depth is redone by the next refine
      c.slab_planned = c.opts.slab_level > 0 ? sl.level == std::min(c.opts.slab_level, g.lfull)
                                             : sl.level == auto_slab_level(g, c.opts.slab_count, g.lfull);
      if (c.fused) {   // the slab-local record table
        c.g.rec_ls = sl.level;
        c.g.rec_z0 = sl.z0;
        c.g.rec_z1 = std::max(sl.z1, sl.z0 + 1);
        lcp_status_t rs = records_setup(c);
        if (rs != LCP_OK) return rs;
      }
    }
    k_node_counts<<<gt, 256, 0, c.stream>>>(g, level, max_depth, F, nF, c.nref.as<int8_t>(), sl, c.cnt.as<int64_t>());
    ++c.n_launch;
    CK(exclusive_scan_i64(c, c.cnt.as<int64_t>(), c.offs.as<int64_t>(), nF, (int64_t*)(dcnt + 1)));
    CK(cudaMemcpyAsync(c.h_counters, dcnt, sizeof(int64_t) * 16, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    int64_t total = c.h_counters[1];
    if (keep) c.n_recs += nF;
    c.level_nodes.push_back(nF);
    c.level_refined.push_back(c.h_counters[12]);
    for (int q = 0; q < 4; ++q) c.level_case[q].push_back(c.h_counters[8 + q]);
    if (level < max_depth) {
      CK(c.front[cur ^ 1].ensure(sizeof(uint64_t) * std::max<int64_t>(total, 1)));
      k_emit<<<gt, 256, 0, c.stream>>>(g, level, max_depth, F, nF, c.nref.as<int8_t>(), c.offs.as<int64_t>(), sl,
                                       c.front[cur ^ 1].as<uint64_t>(), nullptr);
      ++c.n_launch;
      cur ^= 1;
      nF = total;
    } else {
      CK(c.leaves.ensure(sizeof(int64_t) * std::max<int64_t>(total, 1)));
      if (h >= 2) {
        const int64_t nchunk = std::max<int64_t>(1, ((int64_t)1 << (3 * h)) / EMIT_CHUNK);
        k_emit_cells<<<(unsigned)std::min<int64_t>(nF * nchunk, 148 * 16), 256, 0, c.stream>>>(
            g, level, F, nF, c.nref.as<int8_t>(), c.offs.as<int64_t>(), sl, nchunk, c.leaves.as<int64_t>());
      } else {
        k_emit<<<gt, 256, 0, c.stream>>>(g, level, max_depth, F, nF, c.nref.as<int8_t>(), c.offs.as<int64_t>(), sl,
                                         nullptr, c.leaves.as<int64_t>());
      }
      ++c.n_launch;
      c.n_leaves = total;
      nF = 0;
    }
    CK(cudaGetLastError());
  }
  cudaEventRecord(e1, c.stream);
  CK(cudaStreamSynchronize(c.stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  c.t.refine_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
#undef CK
  return check_device_errors(c);
}

}  // namespace lcp
