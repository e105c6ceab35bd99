// common.cuh -- device helpers shared by the liblcp.so kernels (sm_100a).
//
// Nothing here is shared with oracle/: the oracle is an independent C
// implementation of the same paper passages.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lcp.h"

namespace lcp {

constexpr int WARP = 32;
constexpr double SQRT2 = 1.4142135623730951;
constexpr double SQRT5 = 2.23606797749979;

// GP prior (Matern-5/2 per BASELINE c4/c5).
struct KernParams {
  int kind;          // LCP_K_SE / LCP_K_MATERN52
  double var;        // sigma_f^2
  double inv_ls[3];  // 1 / l_d  (also the k-NN metric weights, R2)
  double nugget;     // sigma_n^2
  double m0;         // prior mean
};

// Grid and bucket geometry (R3, R23).
struct Geom {
  double lo[3];
  double h[3];      // cell size (hi - lo) / cells
  double sB[3];     // bucket side bs * h
  int cells[3];
  int nb[3];        // buckets per axis
  int bs;           // cells per bucket side (power of two)
  int bs_log2;
  int lfull;        // 2^lfull >= max cells
  int nbuckets;
  int h_full;
  // record table of the refine-time brick pass (SURVEY §8(e) slab-local memory): the
  // level-rec_ls nodes with z index in [rec_z0, rec_z1) (the rank's z-slab; rec_ls = 0,
  // [0, 1) = the whole virtual cube) -- see rec_index()
  int rec_ls, rec_z0, rec_z1;
};

__device__ __forceinline__ double kern_from_r2(const KernParams& p, double r2) {
  if (p.kind == LCP_K_SE) return p.var * exp(-0.5 * r2);
  double r = sqrt(r2);
  double s = SQRT5 * r;
  return p.var * (1.0 + s + (5.0 / 3.0) * r2) * exp(-s);
}

__device__ __forceinline__ double kern_r2(const KernParams& p, double dx, double dy, double dz) {
  double tx = dx * p.inv_ls[0], ty = dy * p.inv_ls[1], tz = dz * p.inv_ls[2];
  return tx * tx + ty * ty + tz * tz;
}

// k-NN metric of R2, evaluated left to right with no FMA contraction so that
// the selected sets are reproducible bit for bit.
__device__ __forceinline__ double knn_d2(const KernParams& p, const double* x, const double* c) {
  double t0 = __dmul_rn(__dsub_rn(x[0], c[0]), p.inv_ls[0]);
  double t1 = __dmul_rn(__dsub_rn(x[1], c[1]), p.inv_ls[1]);
  double t2 = __dmul_rn(__dsub_rn(x[2], c[2]), p.inv_ls[2]);
  return __dadd_rn(__dadd_rn(__dmul_rn(t0, t0), __dmul_rn(t1, t1)), __dmul_rn(t2, t2));
}

// vertex (i,j,k) -> position lo + i h (no contraction)
__device__ __forceinline__ double vpos(const Geom& g, int d, int64_t i) {
  return __dadd_rn(g.lo[d], __dmul_rn((double)i, g.h[d]));
}

__device__ __forceinline__ int clampi(long long v, int lo, int hi) {
  return (int)(v < lo ? lo : (v > hi ? hi : v));
}

// R3: point -> bucket floor((x - lo) / sB) clamped.
__device__ __forceinline__ int point_bucket_axis(const Geom& g, int d, double x) {
  double t = floor(__ddiv_rn(__dsub_rn(x, g.lo[d]), g.sB[d]));
  t = t < -1.0 ? -1.0 : (t > 2e9 ? 2e9 : t);
  return clampi((long long)t, 0, g.nb[d] - 1);
}
__device__ __forceinline__ int cell_axis(const Geom& g, int d, double x) {
  double t = floor(__ddiv_rn(__dsub_rn(x, g.lo[d]), g.h[d]));
  t = t < -1.0 ? -1.0 : (t > 2e9 ? 2e9 : t);
  return clampi((long long)t, 0, g.cells[d] - 1);
}
// R3: vertex / cell index -> bucket
__device__ __forceinline__ int vbucket_axis(const Geom& g, int d, int64_t i) {
  int64_t b = i >> g.bs_log2;
  return (int)(b < g.nb[d] - 1 ? b : g.nb[d] - 1);
}
__device__ __forceinline__ int bucket_id(const Geom& g, int bx, int by, int bz) {
  return bx + g.nb[0] * (by + g.nb[1] * bz);
}
__device__ __forceinline__ void cell_ijk(const Geom& g, int64_t cell, int& i, int& j, int& k) {
  int64_t nx = g.cells[0], ny = g.cells[1];
  i = (int)(cell % nx);
  int64_t r = cell / nx;
  j = (int)(r % ny);
  k = (int)(r / ny);
}
__device__ __forceinline__ int cell_bucket(const Geom& g, int64_t cell) {
  int i, j, k;
  cell_ijk(g, cell, i, j, k);
  return bucket_id(g, vbucket_axis(g, 0, i), vbucket_axis(g, 1, j), vbucket_axis(g, 2, k));
}
__device__ __forceinline__ void vertex_ijk(const Geom& g, int64_t v, int& i, int& j, int& k) {
  int64_t nx = g.cells[0] + 1, ny = g.cells[1] + 1;
  i = (int)(v % nx);
  int64_t r = v / nx;
  j = (int)(r % ny);
  k = (int)(r / ny);
}
__device__ __forceinline__ int64_t vertex_id(const Geom& g, int64_t i, int64_t j, int64_t k) {
  return i + (int64_t)(g.cells[0] + 1) * (j + (int64_t)(g.cells[1] + 1) * k);
}
__device__ __forceinline__ int vertex_bucket(const Geom& g, int64_t v) {
  int i, j, k;
  vertex_ijk(g, v, i, j, k);
  return bucket_id(g, vbucket_axis(g, 0, i), vbucket_axis(g, 1, j), vbucket_axis(g, 2, k));
}

// 3D Morton code, 21 bits per axis, x in the lowest bit (child c = x + 2y + 4z).
__host__ __device__ __forceinline__ uint64_t spread3(uint64_t v) {
  v &= 0x1FFFFF;
  v = (v | (v << 32)) & 0x1F00000000FFFFull;
  v = (v | (v << 16)) & 0x1F0000FF0000FFull;
  v = (v | (v << 8)) & 0x100F00F00F00F00Full;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
__host__ __device__ __forceinline__ uint64_t morton3(uint64_t x, uint64_t y, uint64_t z) {
  return spread3(x) | (spread3(y) << 1) | (spread3(z) << 2);
}

// Slab-local index of cell (ci, cj, ck)'s MC record: the slab's level-rec_ls nodes in
// (k - z0, j, i) order, each node's cells in Morton order (a node's 8^sh cells are
// consecutive, so a 4^3 brick's 64 records stay 64 consecutive slots).  With rec_ls = 0
// this is the cell's Morton code in the virtual 2^lfull cube.
__host__ __device__ __forceinline__ bool rec_in_slab(const Geom& g, int ck) {
  const int nk = ck >> (g.lfull - g.rec_ls);
  return nk >= g.rec_z0 && nk < g.rec_z1;
}
__host__ __device__ __forceinline__ int64_t rec_index(const Geom& g, int ci, int cj, int ck) {
  const int sh = g.lfull - g.rec_ls;
  const uint64_t node = ((uint64_t)((ck >> sh) - g.rec_z0) << (2 * g.rec_ls)) |
                        ((uint64_t)(cj >> sh) << g.rec_ls) | (uint64_t)(ci >> sh);
  return (int64_t)((node << (3 * sh)) | (morton3(ci, cj, ck) & ((1ull << (3 * sh)) - 1)));
}
// records in the table: (z1 - z0) 4^rec_ls nodes x 8^(lfull - rec_ls) cells
__host__ __forceinline__ int64_t rec_count(const Geom& g) {
  return ((int64_t)(g.rec_z1 - g.rec_z0) << (2 * g.rec_ls)) << (3 * (g.lfull - g.rec_ls));
}

// packed node key (i | j << 21 | k << 42)
__host__ __device__ __forceinline__ uint64_t node_key(uint64_t i, uint64_t j, uint64_t k) {
  return i | (j << 21) | (k << 42);
}
__host__ __device__ __forceinline__ void node_unkey(uint64_t key, int& i, int& j, int& k) {
  i = (int)(key & 0x1FFFFF);
  j = (int)((key >> 21) & 0x1FFFFF);
  k = (int)((key >> 42) & 0x1FFFFF);
}

// packed lower triangle, column major: element (i, j), i >= j
__host__ __device__ __forceinline__ int64_t tri_col(int64_t j, int64_t k) {
  return j * k - (j * (j - 1)) / 2;
}
__host__ __device__ __forceinline__ int64_t tri_size(int64_t k) { return k * (k + 1) / 2; }

// L^-1 stored as DMMA A-fragments (the "LA" layout of a bucket block): row
// tile rt (rows 8rt..8rt+7) and k-step js (columns 4js..4js+3), js <= 2rt+1,
// are 32 doubles in lane order lane = 4 (row - 8rt) + (col - 4js), zero above
// the diagonal and beyond k.  A lane of a DMMA.8x8x4 loads element `lane` of
// block (rt, js): conflict-free and without index arithmetic.
__host__ __device__ __forceinline__ int la_nrt(int k) { return (k + 7) >> 3; }
__host__ __device__ __forceinline__ int64_t la_size(int k) {
  int64_t n = la_nrt(k);
  return n * (n + 1) * 32;
}
__host__ __device__ __forceinline__ int64_t la_block(int rt, int js) { return ((int64_t)rt * (rt + 1) + js) * 32; }

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// device-side error flags (OR-ed; checked by the host at sync points)
enum : int { DERR_NUMERIC = 1, DERR_FACTOR = 2, DERR_OVERFLOW = 4, DERR_INPUT = 8 };

}  // namespace lcp
