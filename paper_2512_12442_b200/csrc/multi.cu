// multi.cu -- NEXT-3: the fused multi-isovalue leaf pass.
//
// The paper sweeps the isovalue; c4 runs three.  Alg. 1
// is run once per isovalue -- the vertex marginals are
// isovalue-free and stay cached in ctx.vcache, so only the first refine pays for
// them -- and each isovalue's leaves set bit t of a dense per-cell mask.  The
// union of the leaf sets is compacted in Morton order of the cells (aligned 4^3
// bricks stay contiguous for k_brick_posterior), then ONE posterior + chol8 per
// union cell and ONE sample stream (k_pmc<T>) count the crossings of every
// isovalue (R27).  A cell pruned for isovalue t gets LCP 0 there.
#include <algorithm>
#include <cmath>

#include "ctx.h"

namespace lcp {

constexpr int UNION_THREADS = 256;
constexpr int UNION_PER_THREAD = 4;
constexpr int UNION_TILE = UNION_THREADS * UNION_PER_THREAD;   // Morton codes per block

__device__ __forceinline__ uint32_t compact3(uint64_t v) {
  v &= 0x1249249249249249ull;
  v = (v ^ (v >> 2)) & 0x10C30C30C30C30C3ull;
  v = (v ^ (v >> 4)) & 0x100F00F00F00F00Full;
  v = (v ^ (v >> 8)) & 0x1F0000FF0000FFull;
  v = (v ^ (v >> 16)) & 0x1F00000000FFFFull;
  v = (v ^ (v >> 32)) & 0x1FFFFFull;
  return (uint32_t)v;
}

// bit t of mask[cell] for every leaf of isovalue t (a leaf list holds each cell once)
__global__ void k_mark_leaves(const int64_t* __restrict__ leaves, int64_t n, uint16_t bit, uint16_t* __restrict__ mask) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) mask[leaves[q]] |= bit;
}

// cell id and mask of Morton code mc of the virtual 2^lfull cube (0 if outside the grid)
__device__ __forceinline__ uint16_t union_probe(const Geom& g, const uint16_t* __restrict__ mask, uint64_t mc,
                                                int64_t& cell) {
  const uint32_t x = compact3(mc), y = compact3(mc >> 1), z = compact3(mc >> 2);
  if (x >= (uint32_t)g.cells[0] || y >= (uint32_t)g.cells[1] || z >= (uint32_t)g.cells[2]) return 0;
  cell = (int64_t)x + (int64_t)g.cells[0] * ((int64_t)y + (int64_t)g.cells[1] * z);
  return mask[cell];
}

__global__ void __launch_bounds__(UNION_THREADS) k_union_count(Geom g, const uint16_t* __restrict__ mask,
                                                               uint64_t ncodes, int64_t* __restrict__ cnt) {
  const uint64_t b0 = (uint64_t)blockIdx.x * UNION_TILE;
  int c = 0;
#pragma unroll
  for (int r = 0; r < UNION_PER_THREAD; ++r) {
    const uint64_t mc = b0 + (uint64_t)r * UNION_THREADS + threadIdx.x;
    int64_t cell;
    if (mc < ncodes && union_probe(g, mask, mc, cell)) ++c;
  }
  c = warp_sum(c);
  __shared__ int ws[UNION_THREADS / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < UNION_THREADS / 32; ++w) t += ws[w];
    cnt[blockIdx.x] = t;
  }
}

// Morton-ordered compaction: round r of the block covers codes [b0 + r*256, b0 + (r+1)*256)
__global__ void __launch_bounds__(UNION_THREADS) k_union_emit(Geom g, const uint16_t* __restrict__ mask,
                                                              uint64_t ncodes, const int64_t* __restrict__ offs,
                                                              int64_t* __restrict__ cells_out,
                                                              uint32_t* __restrict__ mask_out) {
  __shared__ int ws[UNION_THREADS / 32];
  const uint64_t b0 = (uint64_t)blockIdx.x * UNION_TILE;
  int64_t o = offs[blockIdx.x];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int r = 0; r < UNION_PER_THREAD; ++r) {
    const uint64_t mc = b0 + (uint64_t)r * UNION_THREADS + threadIdx.x;
    int64_t cell = 0;
    const uint16_t mk = mc < ncodes ? union_probe(g, mask, mc, cell) : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, mk != 0);
    if (lane == 0) ws[wid] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < UNION_THREADS / 32; ++w) {
      before += w < wid ? ws[w] : 0;
      total += ws[w];
    }
    if (mk) {
      const int64_t slot = o + before + __popc(bal & ((1u << lane) - 1u));
      cells_out[slot] = cell;
      mask_out[slot] = mk;
    }
    o += total;
    __syncthreads();
  }
}

lcp_status_t pmc_multi_impl(Ctx& c, const int64_t* cells, int64_t n, const double* thetas, int T,
                            const uint32_t* mask, int64_t N, uint64_t seed, uint32_t iso, float* out,
                            int64_t stride);
cudaError_t launch_scatter(Ctx& c, const int64_t* cells, const float* lcp, int64_t n, float* field);

lcp_status_t run_field_multi_impl(Ctx& c, const double* thetas, int T, double alpha, int max_depth, int64_t N,
                                  uint64_t seed, uint32_t stream, float* fields, int64_t* n_leaf_out,
                                  int64_t* n_union_out) {
  NvtxRange nvtx_("lcp_run_field_multi (T = %d)", T);
  if (!c.fitted) return set_err(c, LCP_ESTATE, "run_field_multi before fit");
  if (T < 1 || T > 16) return set_err(c, LCP_EINVAL, "run_field_multi: need 1 <= n_iso <= 16");
  cudaError_t e;
#define CK(x)                                        \
  do {                                               \
    e = (x);                                         \
    if (e != cudaSuccess) return cuda_err(c, e, #x); \
  } while (0)
  const Geom& g = c.g;
  if (g.lfull > 11) return set_err(c, LCP_EINVAL, "run_field_multi: grids above 2048 cells per axis");
  const int64_t ncell = (int64_t)g.cells[0] * g.cells[1] * g.cells[2];
  CK(c.cellmask.ensure(sizeof(uint16_t) * ncell));
  uint16_t* cm = c.cellmask.as<uint16_t>();
  CK(cudaMemsetAsync(cm, 0, sizeof(uint16_t) * ncell, c.stream));
  double refine_ms = 0.0;
  for (int t = 0; t < T; ++t) {
    lcp_status_t st = refine_impl(c, thetas[t], alpha, max_depth);
    if (st != LCP_OK) return st;
    refine_ms += c.t.refine_ms;
    if (n_leaf_out) n_leaf_out[t] = c.n_leaves;
    if (c.n_leaves > 0) {
      k_mark_leaves<<<(unsigned)((c.n_leaves + 255) / 256), 256, 0, c.stream>>>(c.leaves.as<int64_t>(), c.n_leaves,
                                                                               (uint16_t)(1u << t), cm);
      ++c.n_launch;
    }
  }
  // union in Morton order of the virtual cube
  cudaEventRecord(c.ev[6], c.stream);
  const uint64_t ncodes = (uint64_t)1 << (3 * g.lfull);
  const int64_t nblk = (int64_t)((ncodes + UNION_TILE - 1) / UNION_TILE);
  CK(c.cnt.ensure(sizeof(int64_t) * nblk));
  CK(c.offs.ensure(sizeof(int64_t) * nblk));
  CK(c.counters.ensure(sizeof(unsigned long long) * 16));
  unsigned long long* dcnt = c.counters.as<unsigned long long>();
  k_union_count<<<(unsigned)nblk, UNION_THREADS, 0, c.stream>>>(g, cm, ncodes, c.cnt.as<int64_t>());
  ++c.n_launch;
  CK(exclusive_scan_i64(c, c.cnt.as<int64_t>(), c.offs.as<int64_t>(), nblk, (int64_t*)(dcnt + 2)));
  CK(cudaMemcpyAsync(c.h_counters + 2, dcnt + 2, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  const int64_t nu = c.h_counters[2];
  if (n_union_out) *n_union_out = nu;
  CK(c.union_cells.ensure(sizeof(int64_t) * std::max<int64_t>(nu, 1)));
  CK(c.union_mask.ensure(sizeof(uint32_t) * std::max<int64_t>(nu, 1)));
  k_union_emit<<<(unsigned)nblk, UNION_THREADS, 0, c.stream>>>(g, cm, ncodes, c.offs.as<int64_t>(),
                                                               c.union_cells.as<int64_t>(),
                                                               c.union_mask.as<uint32_t>());
  ++c.n_launch;
  CK(cudaGetLastError());
  cudaEventRecord(c.ev[7], c.stream);
  CK(c.lcp_tmp.ensure(sizeof(float) * std::max<int64_t>(nu * T, 1)));
  float* lcp = c.lcp_tmp.as<float>();
  lcp_status_t st = pmc_multi_impl(c, c.union_cells.as<int64_t>(), nu, thetas, T, c.union_mask.as<uint32_t>(), N,
                                   seed, stream, lcp, nu);
  if (st != LCP_OK) return st;
  float ums = 0;
  cudaEventElapsedTime(&ums, c.ev[6], c.ev[7]);
  c.t.refine_ms = refine_ms + ums;
  c.n_union = nu;
  cudaEventRecord(c.ev[4], c.stream);
  for (int t = 0; t < T; ++t)
    CK(launch_scatter(c, c.union_cells.as<int64_t>(), lcp + (int64_t)t * nu, nu, fields + (int64_t)t * ncell));
  cudaEventRecord(c.ev[5], c.stream);
#undef CK
  return LCP_OK;
}

}  // namespace lcp
