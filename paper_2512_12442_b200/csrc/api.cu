// api.cu -- the C ABI of liblcp.so (include/lcp.h): argument checks, host <->
// device marshalling, error mapping.  All arithmetic happens in the kernels of
// fit.cu, octree.cu, marginals.cu, pmc.cu and scan.cu.
#include <cstdio>
#include <cstring>
#include <new>

#include "ctx.h"

namespace lcp {

lcp_status_t set_err(Ctx& c, lcp_status_t st, const std::string& msg) {
  c.err = msg;
  return st;
}

lcp_status_t cuda_err(Ctx& c, cudaError_t e, const char* where) {
  c.err = std::string(where) + ": " + cudaGetErrorString(e);
  cudaGetLastError();   // a failed launch's error belongs to this call, not to the next one
  return e == cudaErrorMemoryAllocation ? LCP_ENOMEM : LCP_ECUDA;
}

lcp_status_t check_device_errors(Ctx& c) {
  int h = 0;
  cudaError_t e = cudaMemcpyAsync(&h, c.derr.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
  if (e != cudaSuccess) return cuda_err(c, e, "device error check");
  if (h != 0) {
    // reported once: the flags belong to the call that raised them, not to later calls
    e = cudaMemsetAsync(c.derr.p, 0, sizeof(int), c.stream);
    if (e != cudaSuccess) return cuda_err(c, e, "device error reset");
  }
  if (h & DERR_INPUT) return set_err(c, LCP_EINVAL, "non-finite input (observation coordinate or value, or an A_M entry)");
  if (h & DERR_FACTOR) return set_err(c, LCP_EFACTOR, "a bucket covariance K_y is not PD after jitter");
  if (h & DERR_NUMERIC) return set_err(c, LCP_ENUMERIC, "posterior variance below -1e-8 sigma_f^2");
  if (h & DERR_OVERFLOW) return set_err(c, LCP_EINVAL, "cell or bucket id out of range");
  return LCP_OK;
}

cudaError_t launch_scatter(Ctx& c, const int64_t* cells, const float* lcp, int64_t n, float* field);

__global__ void k_expand_post(const double* __restrict__ post, int64_t n, double* __restrict__ mu,
                              double* __restrict__ cov) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const double* r = post + 44 * q;
  for (int c = 0; c < 8; ++c) mu[8 * q + c] = r[c];
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b <= a; ++b) {
      double v = r[8 + a * (a + 1) / 2 + b];
      cov[64 * q + 8 * a + b] = v;
      cov[64 * q + 8 * b + a] = v;
    }
}

__global__ void k_point_bucket(Geom g, const double* __restrict__ xyz, int64_t n, int32_t* __restrict__ bkt) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  bkt[q] = bucket_id(g, point_bucket_axis(g, 0, xyz[3 * q]), point_bucket_axis(g, 1, xyz[3 * q + 1]),
                     point_bucket_axis(g, 2, xyz[3 * q + 2]));
}

// caller-given bucket ids: copy, with ids outside [0, nbuckets) flagged and clamped to 0
__global__ void k_check_buckets(const int32_t* __restrict__ in, int64_t n, int32_t nbuckets, int32_t* __restrict__ out,
                                int* __restrict__ derr) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  int32_t b = in[q];
  if (b < 0 || b >= nbuckets) {
    atomicOr(derr, DERR_OVERFLOW);
    b = 0;
  }
  out[q] = b;
}

__global__ void k_gather_sorted(const int32_t* __restrict__ bkt, const int64_t* __restrict__ perm, int64_t n,
                                int32_t* __restrict__ out) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) out[q] = bkt[perm[q]];
}

lcp_status_t point_marginals_impl(Ctx& c, const double* xyz, int64_t n, const int32_t* bkt_in, double* mu,
                                  double* var) {
  if (!c.fitted) return set_err(c, LCP_ESTATE, "point marginals before fit");
  if (n <= 0) return LCP_OK;
  cudaError_t e;
#define CK(x)                                        \
  do {                                               \
    e = (x);                                         \
    if (e != cudaSuccess) return cuda_err(c, e, #x); \
  } while (0)
  CK(c.cell_bucket.ensure(sizeof(int32_t) * 2 * n));
  CK(c.perm.ensure(sizeof(int64_t) * n));
  int32_t* bkt = c.cell_bucket.as<int32_t>();
  unsigned gr = (unsigned)((n + 255) / 256);
  if (bkt_in) {
    k_check_buckets<<<gr, 256, 0, c.stream>>>(bkt_in, n, c.g.nbuckets, bkt, c.derr.as<int>());
    ++c.n_launch;
  } else {
    k_point_bucket<<<gr, 256, 0, c.stream>>>(c.g, xyz, n, bkt);
    ++c.n_launch;
  }
  CK(group_by_bucket(c, bkt, n, c.perm.as<int64_t>()));
  k_gather_sorted<<<gr, 256, 0, c.stream>>>(bkt, c.perm.as<int64_t>(), n, bkt + n);
  ++c.n_launch;
  CK(launch_marginals(c, Q_POINT, c.perm.as<int64_t>(), bkt + n, n, xyz, mu, var, 1, nullptr));
#undef CK
  return check_device_errors(c);
}

}  // namespace lcp

using namespace lcp;

#define CTX_GUARD(ctx)                                              \
  if (!(ctx)) return LCP_EINVAL;                                    \
  Ctx& c = (ctx)->c;                                                \
  {                                                                 \
    cudaError_t _e = cudaSetDevice(c.device);                       \
    if (_e != cudaSuccess) return cuda_err(c, _e, "cudaSetDevice"); \
  }

extern "C" {

lcp_status_t lcp_create(int32_t device, void* cuda_stream, lcp_ctx_t** out) {
  if (!out) return LCP_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0 || device < 0 || device >= ndev) {
    cudaGetLastError();
    return LCP_ECUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) return LCP_ECUDA;
  lcp_ctx_t* h = new (std::nothrow) lcp_ctx_t();
  if (!h) return LCP_ENOMEM;
  Ctx& c = h->c;
  c.device = device;
  cudaDeviceGetAttribute(&c.sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cuda_stream) {
    c.stream = (cudaStream_t)cuda_stream;
    c.own_stream = false;
  } else {
    if (cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete h;
      return LCP_ECUDA;
    }
    c.own_stream = true;
  }
  if (c.derr.ensure(sizeof(int) * 4) != cudaSuccess) {
    delete h;
    return LCP_ENOMEM;
  }
  cudaMemsetAsync(c.derr.p, 0, sizeof(int) * 4, c.stream);
  if (cudaMallocHost(&c.h_counters, sizeof(int64_t) * 16) != cudaSuccess) {
    c.h_counters = nullptr;
    c.derr.release();
    delete h;
    return LCP_ENOMEM;
  }
  for (int i = 0; i < 8; ++i) cudaEventCreate(&c.ev[i]);
  c.ev_init = true;
  *out = h;
  return LCP_OK;
}

void lcp_destroy(lcp_ctx_t* ctx) {
  if (!ctx) return;
  Ctx& c = ctx->c;
  cudaSetDevice(c.device);
  cudaStreamSynchronize(c.stream);
  DevBuf* bufs[] = {&c.X, &c.y, &c.obs_bucket, &c.bcount, &c.bstart, &c.gcount, &c.goff, &c.obs_by_bucket,
                    &c.S, &c.bdata, &c.fscratch, &c.obs_key, &c.obs_sorted_key, &c.obs_sorted_idx, &c.occ[0], &c.occ[1], &c.occ[2], &c.obs_mu,
                    &c.obs_sd, &c.plo, &c.phi, &c.derr, &c.knn_fail, &c.S_knn, &c.box_cnt, &c.vcache, &c.vstate, &c.front[0],
                    &c.front[1], &c.ncase, &c.nref, &c.np1, &c.np2, &c.nU, &c.cnt, &c.offs, &c.scan_tmp,
                    &c.req, &c.req_sorted, &c.counters, &c.leaves, &c.recs, &c.cell_bucket, &c.brick_key, &c.child_bricks, &c.perm,
                    &c.cells_tmp, &c.post, &c.lcp_tmp, &c.field_tmp,
                    &c.brick_flag, &c.brick_idx, &c.brick_start, &c.vscratch, &c.pmc_counters, &c.crec, &c.brick_done, &c.brick_unit, &c.cellmask, &c.union_cells, &c.union_mask, &c.ext_z, &c.ext_v, &c.sgpr_A};
  for (DevBuf* b : bufs) b->release();
  if (c.h_counters) cudaFreeHost(c.h_counters);
  if (c.ev_init)
    for (int i = 0; i < 8; ++i) cudaEventDestroy(c.ev[i]);
  if (c.own_stream) cudaStreamDestroy(c.stream);
  delete ctx;
}

const char* lcp_last_error(const lcp_ctx_t* ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }

lcp_status_t lcp_fit_local(lcp_ctx_t* ctx, const double* xyz, const double* y, int64_t m, int32_t on_device,
                           const lcp_kernel_t* kernel, int32_t k, const lcp_grid_t* grid, const lcp_opts_t* opts) {
  CTX_GUARD(ctx);
  return fit_impl(c, xyz, y, m, on_device, kernel, k, grid, opts);
}

lcp_status_t lcp_fit_sgpr(lcp_ctx_t* ctx, const double* xyz_M, const double* mu_M, const double* A_M, int64_t m,
                          int32_t on_device, const lcp_kernel_t* kernel, int32_t k, const lcp_grid_t* grid,
                          const lcp_opts_t* opts) {
  CTX_GUARD(ctx);
  if (!A_M) return set_err(c, LCP_EINVAL, "fit_sgpr: null A_M");
  if (m > 60000) return set_err(c, LCP_EINVAL, "fit_sgpr: m > 60000 (A_M would exceed 28 GB)");
  if (k > 1024) return set_err(c, LCP_EINVAL, "fit_sgpr: k > 1024");
  return fit_impl(c, xyz_M, mu_M, m, on_device, kernel, k, grid, opts, A_M);
}

lcp_status_t lcp_octree_refine(lcp_ctx_t* ctx, double isovalue, double threshold, int32_t max_depth,
                               int64_t* n_leaf_out, const int64_t** leaf_cells_dev_out) {
  CTX_GUARD(ctx);
  lcp_status_t st = refine_impl(c, isovalue, threshold, max_depth);
  if (st != LCP_OK) return st;
  if (n_leaf_out) *n_leaf_out = c.n_leaves;
  if (leaf_cells_dev_out) *leaf_cells_dev_out = c.leaves.as<int64_t>();
  return LCP_OK;
}

lcp_status_t lcp_pmc_cells(lcp_ctx_t* ctx, const int64_t* cells, int64_t n_cells, int32_t cells_on_device,
                           double isovalue, int64_t n_samples, uint64_t seed, uint32_t iso_index, float* lcp_out,
                           int32_t out_on_device) {
  CTX_GUARD(ctx);
  if (n_cells < 0 || (n_cells > 0 && (!cells || !lcp_out))) return set_err(c, LCP_EINVAL, "pmc: bad arguments");
  if (!c.fitted) return set_err(c, LCP_ESTATE, "pmc before fit");
  if (n_cells == 0) return LCP_OK;
  cudaError_t e;
  const int64_t* dcells = cells;
  if (!cells_on_device) {
    int64_t ncell = (int64_t)c.g.cells[0] * c.g.cells[1] * c.g.cells[2];
    for (int64_t q = 0; q < n_cells; ++q)
      if (cells[q] < 0 || cells[q] >= ncell) return set_err(c, LCP_EINVAL, "pmc: cell id out of range");
    if ((e = c.cells_tmp.ensure(sizeof(int64_t) * n_cells)) != cudaSuccess) return cuda_err(c, e, "alloc");
    if ((e = cudaMemcpyAsync(c.cells_tmp.p, cells, sizeof(int64_t) * n_cells, cudaMemcpyHostToDevice, c.stream)) !=
        cudaSuccess)
      return cuda_err(c, e, "copy cells");
    dcells = c.cells_tmp.as<int64_t>();
  }
  float* dout = lcp_out;
  if (!out_on_device) {
    if ((e = c.lcp_tmp.ensure(sizeof(float) * n_cells)) != cudaSuccess) return cuda_err(c, e, "alloc");
    dout = c.lcp_tmp.as<float>();
  }
  lcp_status_t st = pmc_impl(c, dcells, n_cells, isovalue, n_samples, seed, iso_index, dout);
  if (st != LCP_OK) return st;
  if (!out_on_device) {
    if ((e = cudaMemcpyAsync(lcp_out, dout, sizeof(float) * n_cells, cudaMemcpyDeviceToHost, c.stream)) !=
        cudaSuccess)
      return cuda_err(c, e, "copy lcp");
    if ((e = cudaStreamSynchronize(c.stream)) != cudaSuccess) return cuda_err(c, e, "sync");
  }
  return LCP_OK;
}

lcp_status_t lcp_scatter_field(lcp_ctx_t* ctx, const int64_t* cells_dev, const float* lcp_dev, int64_t n,
                               float* field_dev) {
  CTX_GUARD(ctx);
  if (!c.fitted) return set_err(c, LCP_ESTATE, "scatter before fit");
  if (!field_dev || n < 0 || (n > 0 && (!cells_dev || !lcp_dev))) return set_err(c, LCP_EINVAL, "scatter: bad args");
  cudaError_t e = launch_scatter(c, cells_dev, lcp_dev, n, field_dev);
  return e == cudaSuccess ? LCP_OK : cuda_err(c, e, "scatter");
}

lcp_status_t lcp_run_field(lcp_ctx_t* ctx, double isovalue, double threshold, int32_t max_depth,
                           int64_t n_samples, uint64_t seed, uint32_t iso_index, float* field, int32_t out_on_device,
                           int64_t* n_leaf_out) {
  CTX_GUARD(ctx);
  if (!field) return set_err(c, LCP_EINVAL, "run_field: null field");
  lcp_status_t st = refine_impl(c, isovalue, threshold, max_depth);
  if (st != LCP_OK) return st;
  if (n_leaf_out) *n_leaf_out = c.n_leaves;
  cudaError_t e;
  int64_t n = c.n_leaves;
  if ((e = c.lcp_tmp.ensure(sizeof(float) * std::max<int64_t>(n, 1))) != cudaSuccess) return cuda_err(c, e, "alloc");
  st = pmc_impl(c, c.leaves.as<int64_t>(), n, isovalue, n_samples, seed, iso_index, c.lcp_tmp.as<float>());
  if (st != LCP_OK) return st;
  int64_t ncell = (int64_t)c.g.cells[0] * c.g.cells[1] * c.g.cells[2];
  float* dfield = field;
  if (!out_on_device) {
    if ((e = c.field_tmp.ensure(sizeof(float) * ncell)) != cudaSuccess) return cuda_err(c, e, "alloc");
    dfield = c.field_tmp.as<float>();
  }
  cudaEventRecord(c.ev[4], c.stream);
  if ((e = launch_scatter(c, c.leaves.as<int64_t>(), c.lcp_tmp.as<float>(), n, dfield)) != cudaSuccess)
    return cuda_err(c, e, "scatter");
  cudaEventRecord(c.ev[5], c.stream);
  if (!out_on_device) {
    if ((e = cudaMemcpyAsync(field, dfield, sizeof(float) * ncell, cudaMemcpyDeviceToHost, c.stream)) != cudaSuccess)
      return cuda_err(c, e, "copy field");
  }
  if ((e = cudaStreamSynchronize(c.stream)) != cudaSuccess) return cuda_err(c, e, "sync");
  float ms = 0;
  cudaEventElapsedTime(&ms, c.ev[4], c.ev[5]);
  c.t.scatter_ms = ms;
  return LCP_OK;
}

lcp_status_t lcp_pmc_cells_multi(lcp_ctx_t* ctx, const int64_t* cells_dev, int64_t n_cells, const double* isovalues,
                                 int32_t n_iso, const uint32_t* mask_dev, int64_t n_samples, uint64_t seed,
                                 uint32_t stream, float* lcp_dev) {
  CTX_GUARD(ctx);
  if (n_cells < 0 || !isovalues || (n_cells > 0 && (!cells_dev || !lcp_dev)))
    return set_err(c, LCP_EINVAL, "pmc_multi: bad arguments");
  return pmc_multi_impl(c, cells_dev, n_cells, isovalues, n_iso, mask_dev, n_samples, seed, stream, lcp_dev,
                        n_cells);
}

lcp_status_t lcp_run_field_multi(lcp_ctx_t* ctx, const double* isovalues, int32_t n_iso, double threshold,
                                 int32_t max_depth, int64_t n_samples, uint64_t seed, uint32_t stream,
                                 float* fields, int32_t out_on_device, int64_t* n_leaf_out, int64_t* n_union_out) {
  CTX_GUARD(ctx);
  if (!fields || !isovalues) return set_err(c, LCP_EINVAL, "run_field_multi: null pointer");
  if (n_iso < 1 || n_iso > 16) return set_err(c, LCP_EINVAL, "run_field_multi: need 1 <= n_iso <= 16");
  cudaError_t e;
  const int64_t ncell = (int64_t)c.g.cells[0] * c.g.cells[1] * c.g.cells[2];
  float* dfields = fields;
  if (!out_on_device) {
    if ((e = c.field_tmp.ensure(sizeof(float) * ncell * n_iso)) != cudaSuccess) return cuda_err(c, e, "alloc");
    dfields = c.field_tmp.as<float>();
  }
  lcp_status_t st = run_field_multi_impl(c, isovalues, n_iso, threshold, max_depth, n_samples, seed, stream,
                                         dfields, n_leaf_out, n_union_out);
  if (st != LCP_OK) return st;
  if (!out_on_device) {
    if ((e = cudaMemcpyAsync(fields, dfields, sizeof(float) * ncell * n_iso, cudaMemcpyDeviceToHost, c.stream)) !=
        cudaSuccess)
      return cuda_err(c, e, "copy fields");
  }
  if ((e = cudaStreamSynchronize(c.stream)) != cudaSuccess) return cuda_err(c, e, "sync");
  float ms = 0;
  cudaEventElapsedTime(&ms, c.ev[4], c.ev[5]);
  c.t.scatter_ms = ms;
  return check_device_errors(c);
}

lcp_status_t lcp_union_cells(lcp_ctx_t* ctx, int64_t* n_out, const int64_t** cells_dev_out,
                             const uint32_t** mask_dev_out) {
  CTX_GUARD(ctx);
  if (!n_out || !cells_dev_out || !mask_dev_out) return set_err(c, LCP_EINVAL, "union_cells: null output");
  *n_out = c.n_union;
  *cells_dev_out = c.union_cells.as<int64_t>();
  *mask_dev_out = c.union_mask.as<uint32_t>();
  return LCP_OK;
}

lcp_status_t lcp_set_level_field(lcp_ctx_t* ctx, uint8_t* level_dev) {
  CTX_GUARD(ctx);
  c.level_field = level_dev;
  return LCP_OK;
}

lcp_status_t lcp_node_records(lcp_ctx_t* ctx, int64_t* n_out, const lcp_node_rec_t** recs_dev_out) {
  CTX_GUARD(ctx);
  if (!n_out || !recs_dev_out) return set_err(c, LCP_EINVAL, "node_records: null output");
  *n_out = c.n_recs;
  *recs_dev_out = c.recs.as<lcp_node_rec_t>();
  return LCP_OK;
}

lcp_status_t lcp_cell_posterior(lcp_ctx_t* ctx, const int64_t* cells_dev, int64_t n, double* mu_dev,
                                double* cov_dev) {
  CTX_GUARD(ctx);
  if (!c.fitted) return set_err(c, LCP_ESTATE, "posterior before fit");
  if (n <= 0) return LCP_OK;
  cudaError_t e;
  if ((e = c.post.ensure(sizeof(double) * 44 * n)) != cudaSuccess) return cuda_err(c, e, "alloc");
  lcp_status_t st = posterior_impl(c, cells_dev, n, c.post.as<double>());
  if (st != LCP_OK) return st;
  k_expand_post<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(c.post.as<double>(), n, mu_dev, cov_dev);
  ++c.n_launch;
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_err(c, e, "expand");
  return check_device_errors(c);
}

lcp_status_t lcp_point_marginals(lcp_ctx_t* ctx, const double* xyz_dev, int64_t n, const int32_t* bucket_dev,
                                 double* mu_dev, double* var_dev) {
  CTX_GUARD(ctx);
  return point_marginals_impl(c, xyz_dev, n, bucket_dev, mu_dev, var_dev);
}

lcp_status_t lcp_bucket_sets(lcp_ctx_t* ctx, int32_t* sets_dev) {
  CTX_GUARD(ctx);
  if (!c.fitted) return set_err(c, LCP_ESTATE, "bucket_sets before fit");
  cudaError_t e = cudaMemcpyAsync(sets_dev, c.S.p, sizeof(int32_t) * (size_t)c.g.nbuckets * c.k,
                                  cudaMemcpyDeviceToDevice, c.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
  return e == cudaSuccess ? LCP_OK : cuda_err(c, e, "bucket_sets");
}

lcp_status_t lcp_get_info(lcp_ctx_t* ctx, lcp_info_t* out) {
  CTX_GUARD(ctx);
  if (!out) return LCP_EINVAL;
  std::memset(out, 0, sizeof(*out));
  out->m = c.m;
  out->k = c.k;
  out->nbuckets = c.g.nbuckets;
  for (int d = 0; d < 3; ++d) out->nb[d] = c.g.nb[d];
  out->lfull = c.g.lfull;
  out->bucket_side = c.g.bs;
  out->device = c.device;
  return c.fitted ? LCP_OK : set_err(c, LCP_ESTATE, "info before fit");
}

lcp_status_t lcp_stats_json(lcp_ctx_t* ctx, char* buf, size_t cap) {
  CTX_GUARD(ctx);
  if (!buf || cap == 0) return LCP_EINVAL;
  std::string s = "{";
  char tmp[1024];
  std::snprintf(tmp, sizeof tmp,
                "\"fit_ms\": %.6f, \"refine_ms\": %.6f, \"posterior_ms\": %.6f, \"chol_ms\": %.6f, \"mc_ms\": %.6f, "
                "\"scatter_ms\": %.6f, \"leaves\": %lld, \"pmc_cells\": %lld, \"pmc_samples\": %lld, "
                "\"vertex_marginals\": %lld, \"knn_fallbacks\": %d, \"nbuckets\": %d, \"k\": %d, \"m\": %lld, "
                "\"launches\": %lld, \"brick_runs\": %lld, \"pmc_phase2_samples\": %lld, \"brick_pass_ms\": %.6f, "
                "\"fused\": %d, \"pmc_used_records\": %d, \"capped_buckets\": %d, \"max_set\": %d",
                c.t.fit_ms, c.t.refine_ms, c.t.posterior_ms, c.t.chol_ms, c.t.mc_ms, c.t.scatter_ms,
                (long long)c.n_leaves, (long long)c.last_pmc_cells, (long long)c.last_pmc_samples,
                (long long)c.last_requests, c.knn_fallbacks, c.g.nbuckets, c.k, (long long)c.m,
                (long long)c.n_launch, (long long)c.last_brick_runs,
                (long long)c.last_pmc_phase2, c.t.brick_ms, c.fused ? 1 : 0, c.last_pmc_records ? 1 : 0, c.n_capped,
                c.max_set);
  s += tmp;
  auto arr = [&](const char* name, const std::vector<int64_t>& v) {
    s += ", \"";
    s += name;
    s += "\": [";
    for (size_t i = 0; i < v.size(); ++i) {
      if (i) s += ", ";
      s += std::to_string(v[i]);
    }
    s += "]";
  };
  arr("level_nodes", c.level_nodes);
  arr("level_refined", c.level_refined);
  arr("level_case0", c.level_case[0]);
  arr("level_case1", c.level_case[1]);
  arr("level_case2", c.level_case[2]);
  arr("level_case3", c.level_case[3]);
  if (c.opts.slab_count > 1) {   // the z-slab plan (identical on every rank)
    const int64_t side = (int64_t)1 << (c.g.lfull - c.slab_L);
    std::vector<int64_t> cuts(c.slab_cuts.begin(), c.slab_cuts.end()), ccuts;
    for (int z : c.slab_cuts) ccuts.push_back(std::min<int64_t>((int64_t)z * side, c.g.cells[2]));
    std::snprintf(tmp, sizeof tmp,
                  ", \"slab\": {\"rank\": %d, \"count\": %d, \"level\": %d, \"layers\": %d, \"z0\": %d, "
                  "\"z1\": %d, \"planned\": %d, \"records_ready\": %d, \"record_cells\": %lld",
                  c.opts.slab_rank, c.opts.slab_count, c.slab_L, c.slab_nz, c.slab_z0, c.slab_z1,
                  c.slab_planned ? 1 : 0, c.rec_ready ? 1 : 0, (long long)(c.rec_ready ? rec_count(c.g) : 0));
    s += tmp;
    arr("layer_cuts", cuts);
    arr("cell_z_cuts", ccuts);
    arr("weights", c.slab_w);
    s += "}";
  }
  s += "}";
  if (s.size() + 1 > cap) return set_err(c, LCP_EINVAL, "stats_json: buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return LCP_OK;
}

lcp_status_t lcp_fit_shard_buffers(lcp_ctx_t* ctx, void** bdata_dev, int64_t* bdata_chunk_bytes, void** sets_dev,
                                   int64_t* sets_chunk_bytes) {
  CTX_GUARD(ctx);
  if (!bdata_dev || !bdata_chunk_bytes || !sets_dev || !sets_chunk_bytes) return LCP_EINVAL;
  if (!c.fit_pending) return set_err(c, LCP_ESTATE, "fit_shard_buffers: no sharded fit pending");
  *bdata_dev = c.bdata.p;
  *bdata_chunk_bytes = (int64_t)sizeof(double) * c.bstride * c.shard_per;
  *sets_dev = c.S.p;
  *sets_chunk_bytes = (int64_t)sizeof(int32_t) * c.k * c.shard_per;
  return LCP_OK;
}

lcp_status_t lcp_fit_finish(lcp_ctx_t* ctx) {
  CTX_GUARD(ctx);
  if (!c.fit_pending) return set_err(c, LCP_ESTATE, "fit_finish: no sharded fit pending");
  return fit_finish_impl(c);
}

int32_t lcp_slab_auto_level(const lcp_grid_t* grid, int32_t slab_count, int32_t max_depth) {
  if (!grid || slab_count < 1 || max_depth < 0) return -1;
  lcp::Geom g{};
  int cmax = 1;
  for (int d = 0; d < 3; ++d) {
    if (grid->cells[d] < 1) return -1;
    g.cells[d] = grid->cells[d];
    cmax = std::max(cmax, grid->cells[d]);
  }
  int lf = 0;
  while ((1 << lf) < cmax) ++lf;
  g.lfull = lf;
  return lcp::auto_slab_level(g, slab_count, std::min(max_depth, lf));
}

lcp_status_t lcp_slab_cuts(const int64_t* weights, int32_t n_layers, int32_t slab_count, int32_t* cuts_out) {
  if (!weights || !cuts_out || n_layers < 1 || slab_count < 1) return LCP_EINVAL;
  std::vector<int64_t> w(weights, weights + n_layers);
  for (int64_t v : w)
    if (v < 0) return LCP_EINVAL;
  std::vector<int> cut = lcp::slab_cuts(w, slab_count);
  for (int r = 0; r <= slab_count; ++r) cuts_out[r] = cut[r];
  return LCP_OK;
}

lcp_status_t lcp_synchronize(lcp_ctx_t* ctx) {
  CTX_GUARD(ctx);
  cudaError_t e = cudaStreamSynchronize(c.stream);
  if (e != cudaSuccess) return cuda_err(c, e, "synchronize");
  return check_device_errors(c);
}

}  // extern "C"
