// scan.cu -- device-wide exclusive scan and group-by-bucket (counting sort).
//
// Used by stream compaction of the octree frontier and by
// the bucket grouping of observations, vertex requests and leaf cells so that
// one CTA stages one bucket's local-GP factor into shared memory.
#include "ctx.h"

namespace lcp {

constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

// block-wide exclusive scan of one value per thread; returns the block total
__device__ int64_t block_exclusive_scan(int64_t v, int64_t* smem_warp, int64_t& excl) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int64_t w = lane < nw ? smem_warp[lane] : 0;
    int64_t s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) smem_warp[lane] = s - w;
    if (lane == 31) smem_warp[32] = s;
  }
  __syncthreads();
  excl = smem_warp[wid] + x - v;
  int64_t total = smem_warp[32];
  __syncthreads();
  return total;
}

__global__ void k_scan_reduce(const int64_t* __restrict__ in, int64_t n, int64_t* __restrict__ bsum) {
  __shared__ int64_t sw[33];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int64_t s = 0;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q)
    if (base + q < n) s += in[base + q];
  int64_t ex;
  int64_t tot = block_exclusive_scan(s, sw, ex);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void k_scan_blocksums(int64_t* __restrict__ bsum, int64_t nb, int64_t* __restrict__ total) {
  __shared__ int64_t sw[33];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < nb ? bsum[i] : 0;
    int64_t ex;
    int64_t tot = block_exclusive_scan(v, sw, ex);
    if (i < nb) bsum[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void k_scan_final(const int64_t* __restrict__ in, int64_t n, const int64_t* __restrict__ bsum,
                             int64_t* __restrict__ out) {
  __shared__ int64_t sw[33];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int64_t v[SCAN_ITEMS];
  int64_t s = 0;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    v[q] = base + q < n ? in[base + q] : 0;
    s += v[q];
  }
  int64_t ex;
  block_exclusive_scan(s, sw, ex);
  int64_t run = bsum[blockIdx.x] + ex;
#pragma unroll
  for (int q = 0; q < SCAN_ITEMS; ++q) {
    if (base + q < n) out[base + q] = run;
    run += v[q];
  }
}

cudaError_t exclusive_scan_i64(Ctx& c, const int64_t* in, int64_t* out, int64_t n, int64_t* total_dev) {
  if (n <= 0) {
    if (total_dev) return cudaMemsetAsync(total_dev, 0, sizeof(int64_t), c.stream);
    return cudaSuccess;
  }
  int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  cudaError_t e = c.scan_tmp.ensure(sizeof(int64_t) * (size_t)nb);
  if (e != cudaSuccess) return e;
  int64_t* bs = c.scan_tmp.as<int64_t>();
  k_scan_reduce<<<(unsigned)nb, SCAN_THREADS, 0, c.stream>>>(in, n, bs);
  ++c.n_launch;
  k_scan_blocksums<<<1, SCAN_THREADS, 0, c.stream>>>(bs, nb, total_dev);
  ++c.n_launch;
  k_scan_final<<<(unsigned)nb, SCAN_THREADS, 0, c.stream>>>(in, n, bs, out);
  ++c.n_launch;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- grouping
__global__ void k_bucket_count(const int32_t* __restrict__ bkt, int64_t n, int64_t* __restrict__ cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int b = bkt[i];
  // warp-aggregated increment: lanes with the same bucket add once
  unsigned same = __match_any_sync(__activemask(), b);
  int leader = __ffs(same) - 1;
  if ((int)(threadIdx.x & 31) == leader) atomicAdd((unsigned long long*)&cnt[b], (unsigned long long)__popc(same));
}

__global__ void k_bucket_scatter(const int32_t* __restrict__ bkt, int64_t n, int64_t* __restrict__ cursor,
                                 int64_t* __restrict__ perm) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int b = bkt[i];
  unsigned same = __match_any_sync(__activemask(), b);
  int lane = threadIdx.x & 31;
  int leader = __ffs(same) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd((unsigned long long*)&cursor[b], (unsigned long long)__popc(same));
  base = __shfl_sync(same, base, leader);
  int rank = __popc(same & ((1u << lane) - 1u));
  perm[base + rank] = i;
}

// perm_out[n]: item indices grouped by bucket (order inside a bucket is
// unspecified; every consumer's result is a function of the item alone).
cudaError_t group_by_bucket(Ctx& c, const int32_t* bucket_of_item, int64_t n, int64_t* perm_out) {
  return group_by_key(c, bucket_of_item, n, c.g.nbuckets, perm_out);
}

// counting sort of items by an int32 key in [0, nkeys) (order within a key unspecified)
cudaError_t group_by_key(Ctx& c, const int32_t* bucket_of_item, int64_t n, int64_t nkeys, int64_t* perm_out) {
  if (n <= 0) return cudaSuccess;
  int64_t nbk = nkeys;
  cudaError_t e = c.gcount.ensure(sizeof(int64_t) * (nbk + 1));
  if (e != cudaSuccess) return e;
  e = c.goff.ensure(sizeof(int64_t) * (nbk + 1));
  if (e != cudaSuccess) return e;
  int64_t* cnt = c.gcount.as<int64_t>();
  int64_t* off = c.goff.as<int64_t>();
  cudaMemsetAsync(cnt, 0, sizeof(int64_t) * nbk, c.stream);
  unsigned grid = (unsigned)((n + 255) / 256);
  k_bucket_count<<<grid, 256, 0, c.stream>>>(bucket_of_item, n, cnt);
  ++c.n_launch;
  e = exclusive_scan_i64(c, cnt, off, nbk, nullptr);
  if (e != cudaSuccess) return e;
  k_bucket_scatter<<<grid, 256, 0, c.stream>>>(bucket_of_item, n, off, perm_out);
  ++c.n_launch;
  return cudaGetLastError();
}

}  // namespace lcp
