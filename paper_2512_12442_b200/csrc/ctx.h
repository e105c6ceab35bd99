// ctx.h -- host-side context of liblcp.so and the internal launch interface.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing without a tool attached

#include "common.cuh"
#include "lcp.h"

namespace lcp {

// grow-only device buffer (allocation happens only when a call needs more)
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = bytes + bytes / 4 + 256;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  // grow keeping the first `used` bytes (stream-ordered copy)
  cudaError_t ensure_keep(size_t bytes, size_t used, cudaStream_t s) {
    if (bytes <= cap) return cudaSuccess;
    size_t want = bytes + bytes / 2 + 256;
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, want);
    if (e != cudaSuccess) return e;
    if (p && used) {
      e = cudaMemcpyAsync(q, p, used, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return e;
      cudaStreamSynchronize(s);
    }
    if (p) cudaFree(p);
    p = q;
    cap = want;
    return cudaSuccess;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <typename T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

// host-side trace range (NVTX) around a phase of a call: visible in Nsight Systems / ncu
// --nvtx timelines; a no-op unless a profiler is attached
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* fmt, int v) {
    char b[64];
    std::snprintf(b, sizeof b, fmt, v);
    nvtxRangePushA(b);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr int64_t BRICK_PASS_CHUNK = (int64_t)1 << 17;   // bricks per brick-pass launch (8.4 M cells)

struct PhaseTimes {
  double fit_ms = 0, refine_ms = 0, posterior_ms = 0, chol_ms = 0, mc_ms = 0, scatter_ms = 0;
  double brick_ms = 0;   // refine-time brick pass (part of refine_ms)
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int sm_count = 148;

  // model (after fit)
  bool fitted = false;
  bool fit_pending = false;  // sharded fit: bucket blocks of the other ranks not exchanged yet
  int shard_per = 0;         // sharded fit: buckets per rank (the last rank's range padded)
  KernParams kp{};
  Geom g{};
  lcp_kernel_t kern{};
  lcp_grid_t grid{};
  lcp_opts_t opts{};
  int64_t m = 0;
  int k = 0;
  int64_t bstride = 0;       // doubles per bucket block [Linv tri(k) | alpha k | Xs 3k], padded to 2
  double kcc[36];            // prior covariance among the 8 corners of a cell (packed lower)

  DevBuf X, y;               // observations, SoA x[m] y[m] z[m] / y[m]
  DevBuf obs_bucket;         // int32 point bucket per obs
  DevBuf bcount, bstart;     // per bucket observation counts / starts (int64)
  DevBuf gcount, goff;       // group_by_bucket scratch (int64)
  DevBuf obs_by_bucket;      // int32 observations grouped by bucket
  DevBuf S;                  // int32 nbuckets x k (ascending)
  DevBuf bdata;              // double nbuckets x bstride
  DevBuf fscratch;           // factor scratch for large k
  DevBuf sgpr_A;             // NEXT-2: A_M (m x m) of an SGPR model
  DevBuf obs_key, obs_sorted_key, obs_sorted_idx;  // Morton keys of the finest cell
  DevBuf occ[3];                 // occupancy bitmaps of nodes at heights 0, 1, 2 (bit per Morton code)
  int occ_heights = 0;           // how many of occ[] are built (0 when the cube is too large)
  DevBuf obs_mu, obs_sd;     // observation marginals (Morton order after fit)
  DevBuf plo, phi;           // per-theta observation tails (Morton order)
  DevBuf derr;               // device error flags (int)
  DevBuf knn_fail;           // int: buckets whose ring search overflowed
  DevBuf S_knn, box_cnt;     // local_mode 2: k-NN sets, beta-box counts per bucket
  int n_capped = 0;          // local_mode 2: buckets whose beta-box exceeded k (took the k-NN set)
  int knn_fallbacks = 0;
  int max_set = 0;            // box mode: largest bucket set
  int64_t n_launch = 0;      // kernels this ctx has launched (cumulative)
  int64_t n_vertices = 0;    // (nx+1)(ny+1)(nz+1)
  int64_t last_requests = 0; // vertex marginals computed by the last refine

  // octree state
  DevBuf vcache;             // double2 (mu, sd) per grid vertex
  DevBuf vstate;             // uint32 bitmask over grid vertices: marginal requested/ready
  bool vcache_valid = false;
  DevBuf front[2];           // uint64 node keys
  DevBuf ncase, nref;        // per node of the level
  DevBuf np1, np2, nU;       // per node of the level (double)
  DevBuf cnt, offs;          // int64 per node: children / leaf counts and offsets
  DevBuf scan_tmp;
  DevBuf req, req_sorted;    // vertex requests
  DevBuf counters;           // int64 device counters
  DevBuf leaves;             // int64 leaf cell ids
  int64_t n_leaves = 0;
  DevBuf recs;               // lcp_node_rec_t
  DevBuf ext_z, ext_v;       // NEXT-1: lattice extremes (z, vertex) per node
  uint8_t* level_field = nullptr;  // NEXT-4: caller-owned per-cell level output (lcp_set_level_field)
  int64_t n_recs = 0;

  // leaf pass scratch
  DevBuf cell_bucket, brick_key, perm, cells_tmp, post, lcp_tmp, field_tmp, child_bricks;
  DevBuf brick_flag, brick_idx, brick_start;
  DevBuf vscratch;               // k_brick_big: per-CTA V scratch (L2-resident)
  // refine-time brick pass (brick.cu k_brick<true>): MC records of every cell of the
  // level-(Lfull-2) frontier bricks, indexed by the cell's Morton code
  bool fused = false;            // enabled for this fit (supported and records fit in HBM)
  bool rec_ready = false;        // the record table of the current slab is allocated and cleared
  DevBuf crec;                   // CellRec per cell of the rank's slab (rec_index, common.cuh)
  DevBuf brick_done;             // uint8 per brick of the slab (rec_index >> 6)
  DevBuf brick_unit;             // uint8 per unit of a brick-pass launch: computed by it
  DevBuf cellmask;               // NEXT-3: uint16 per cell, bit t = leaf of isovalue t
  DevBuf union_cells, union_mask; // NEXT-3: union leaf list (Morton order) and its masks
  int64_t n_union = 0;
  DevBuf pmc_counters;           // [0]: samples finished in phase 2 of k_pmc
  int64_t last_pmc_phase2 = 0;
  bool last_pmc_records = false; // the last pmc read the brick-pass records
  int64_t last_brick_runs = 0;   // brick runs of the last posterior (0: per-cell path)

  // host pinned staging for counters
  int64_t* h_counters = nullptr;

  // z-slab decomposition: placed by the first refine after a fit, from the
  // refined level-slab_L nodes per z-layer (identical on every rank), kept until the next fit
  bool slab_planned = false;
  int slab_L = 0, slab_nz = 0, slab_z0 = 0, slab_z1 = 0;
  std::vector<int64_t> slab_w;   // weights per z-layer of level slab_L
  std::vector<int> slab_cuts;    // slab_count + 1 layer cuts (rank r owns [cuts[r], cuts[r+1]))

  // stats
  PhaseTimes t;
  std::vector<int64_t> level_nodes, level_refined, level_case[4];
  int64_t last_pmc_cells = 0, last_pmc_samples = 0;
  cudaEvent_t ev[8];
  bool ev_init = false;
};

// ---- internal launchers (implemented in the .cu files) ----
cudaError_t exclusive_scan_i64(Ctx& c, const int64_t* in, int64_t* out, int64_t n, int64_t* total_dev);
cudaError_t group_by_bucket(Ctx& c, const int32_t* bucket_of_item, int64_t n, int64_t* perm_out);
cudaError_t group_by_key(Ctx& c, const int32_t* key_of_item, int64_t n, int64_t nkeys, int64_t* perm_out);

lcp_status_t fit_impl(Ctx& c, const double* xyz, const double* y, int64_t m, int on_device,
                      const lcp_kernel_t* kern, int k, const lcp_grid_t* grid, const lcp_opts_t* opts,
                      const double* AM = nullptr);
lcp_status_t fit_finish_impl(Ctx& c);
lcp_status_t refine_impl(Ctx& c, double theta, double alpha, int max_depth);
lcp_status_t pmc_impl(Ctx& c, const int64_t* cells_dev, int64_t n, double theta, int64_t N,
                      uint64_t seed, uint32_t iso, float* out_dev);
lcp_status_t pmc_multi_impl(Ctx& c, const int64_t* cells_dev, int64_t n, const double* thetas, int T,
                            const uint32_t* mask_dev, int64_t N, uint64_t seed, uint32_t stream, float* out_dev,
                            int64_t stride);
lcp_status_t run_field_multi_impl(Ctx& c, const double* thetas, int T, double alpha, int max_depth, int64_t N,
                                  uint64_t seed, uint32_t stream, float* fields_dev, int64_t* n_leaf_out,
                                  int64_t* n_union_out);
lcp_status_t posterior_impl(Ctx& c, const int64_t* cells_dev, int64_t n, double* post_dev);
lcp_status_t point_marginals_impl(Ctx& c, const double* xyz_dev, int64_t n, const int32_t* bkt,
                                  double* mu_dev, double* var_dev);
lcp_status_t check_device_errors(Ctx& c);

// marginals / posterior tile kernels (marginals.cu)
enum QueryMode : int { Q_VERTEX = 0, Q_OBS = 1, Q_POINT = 2 };
cudaError_t launch_marginals(Ctx& c, int mode, const int64_t* items_sorted, const int32_t* item_bucket_sorted,
                             int64_t n, const double* points, double* out_mu, double* out_sd_or_var,
                             int write_var, const int64_t* n_dev);
cudaError_t launch_cell_posterior(Ctx& c, const int64_t* cells, const int64_t* perm,
                                  const int32_t* bkt_sorted, int64_t n, double* post);
bool brick_posterior(Ctx& c, const int64_t* cells, int64_t n, double* post, cudaError_t& err);
bool fused_brick_supported(const Ctx& c);
bool brick_posterior_big(Ctx& c, const int64_t* cells, int64_t n, double* post, cudaError_t& err);
cudaError_t launch_brick_pass(Ctx& c, const uint64_t* bricks, int64_t nb, double* post);
cudaError_t launch_child_bricks(Ctx& c, const uint64_t* F, int64_t nF, int gen, uint64_t* out);
cudaError_t launch_chol8_rec(Ctx& c, const uint64_t* bricks, int64_t nb, const double* post);
lcp_status_t fused_setup(Ctx& c);
lcp_status_t records_setup(Ctx& c);

// z-slab plan (octree.cu; host code, also behind lcp_slab_auto_level / lcp_slab_cuts)
int slab_layers_at(const Geom& g, int L);
int auto_slab_level(const Geom& g, int count, int max_depth);
std::vector<int> slab_cuts(const std::vector<int64_t>& w, int count);

lcp_status_t set_err(Ctx& c, lcp_status_t st, const std::string& msg);
lcp_status_t cuda_err(Ctx& c, cudaError_t e, const char* where);

}  // namespace lcp

struct lcp_ctx {
  lcp::Ctx c;
};
