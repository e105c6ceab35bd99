/*
 * lcp.h -- C ABI of the B200-native level-crossing-probability (LCP) library.
 *
 * Implements the data-parallel hot path of arxiv 2512.12442 ("efficient LCP
 * computation for GP-represented data"; PAPER.md = /root/reference/PAPER.md):
 *   - lcp_fit_local      : bucket-local k-NN GP factors
 *   - lcp_octree_refine  : Alg. 1 octree with the Eq. 4 bound   (a5-a6)
 *   - lcp_pmc_cells      : per-cell posterior + 8x8 Cholesky + Philox MC (a7-a8)
 *   - lcp_scatter_field / lcp_run_field : dense LCP field output (a9)
 * Every step runs in hand-written sm_100a kernels of liblcp.so.  There is no
 * CPU fallback: without a CUDA device every call returns LCP_ECUDA.
 *
 * Conventions: cell size h_d = (hi_d - lo_d) / cells_d; vertex
 * (i,j,k) at lo + (i,j,k) h; cell id = i + nx (j + ny k) (x fastest); corner
 * c = c0 + 2 c1 + 4 c2 of cell (i,j,k) is vertex (i+c0, j+c1, k+c2)
 * (PAPER.md:118-122).  Pointers are plain host or device pointers as stated
 * per argument; "device" pointers must be valid on the ctx's device.
 *
 * Errors: every call returns lcp_status_t; outputs are undefined unless the
 * status is LCP_OK, and lcp_last_error() then holds a message.  No exception
 * or abort crosses the ABI.  Threading: one ctx per device per host thread.
 */
#ifndef LCP_H
#define LCP_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lcp_ctx lcp_ctx_t;   /* opaque; owns all device caches */

typedef enum {
    LCP_OK = 0,
    LCP_EINVAL = 1,    /* bad argument (alpha not in (0,0.5), N < 1, k < 1 or k > m, ...) */
    LCP_ESTATE = 2,    /* refine / pmc before fit */
    LCP_EFACTOR = 3,   /* a bucket K_y not PD even after jitter 1e-10..1e-8 sigma_f^2 (R15) */
    LCP_ENUMERIC = 4,  /* a posterior variance < -1e-8 sigma_f^2 (R16) */
    LCP_ECUDA = 5,     /* CUDA runtime error (incl. no device) */
    LCP_ENOMEM = 6     /* device allocation failed */
} lcp_status_t;

typedef enum { LCP_K_SE = 0, LCP_K_MATERN52 = 1 } lcp_kernel_kind_t;
typedef enum { LCP_FP64 = 0, LCP_FP32 = 1 } lcp_prec_t;

/* GP prior: k(x1,x2) = variance * f(|(x1-x2)/lengthscale|);
 * SE f = exp(-r^2/2); Matern-5/2 f = (1 + sqrt5 r + 5/3 r^2) exp(-sqrt5 r).
 * nugget = observation noise variance sigma_n^2 (R1); prior_mean = m0. */
typedef struct {
    int32_t kind;
    int32_t pad_;
    double variance;
    double lengthscale[3];
    double nugget;
    double prior_mean;
} lcp_kernel_t;

/* target grid: domain [lo, hi], cells[d] cells per axis */
typedef struct {
    double lo[3];
    double hi[3];
    int32_t cells[3];
    int32_t pad_;
} lcp_grid_t;

typedef struct {
    int32_t bucket_log2;   /* bucket grid: 2^bucket_log2 buckets per axis of the virtual cube (R3) */
    int32_t h_full;        /* candidate lattice: all vertices at node heights <= h_full (R6);
                              min(h_full, Lfull) <= 10 */
    int32_t precision;     /* lcp_prec_t of the leaf posterior (R17) */
    int32_t slab_rank;     /* z-slab decomposition: this rank ... */
    int32_t slab_count;    /* ... of slab_count (1 = whole domain).  Every rank evaluates the
                              octree levels 0..slab_level over the whole domain; the first refine
                              after a fit then cuts the z-layers of level slab_level into
                              slab_count contiguous ranges by prefix sums of the refined
                              level-slab_level nodes per layer (identical on every rank, no
                              communication) and keeps the children of layers [z0, z1) only;
                              the cut stands until the next fit (lcp_stats_json "slab") */
    int32_t slab_level;    /* <= 0: automatic -- the shallowest level with >= 2 slab_count
                              z-layers, at most min(max_depth, Lfull - 3); else that level */
    int32_t keep_records;  /* parity tap: keep per-node records of levels < keep_records (0 = none) */
    int32_t extreme_iters; /* NEXT-1 (R26): iterations of the continuous extreme search at nodes
                              coarser than h_full; 0 = lattice only */
    int32_t brick_pass;    /* refine-time brick pass (vertex marginals + MC records of every
                              level-(Lfull-2) frontier brick): 0 = on when supported and the
                              records (208 B per cell) fit in free HBM, -1 = off */
    int32_t local_mode;    /* bucket local sets: 0 = the k nearest observations to the bucket
                              centre (R2, BASELINE); 1 = every observation inside the bucket box
                              enlarged by beta * lengthscale per axis (R28, PAPER.md:197-199:
                              the paper's M' of the level-bucket_log2 node), at most k of them
                              (EINVAL otherwise), padded to k internally; 2 = as 1, with the
                              |M'| cap k: a bucket whose box holds more than k takes its k-NN
                              set instead (R28b; lcp_stats_json "capped_buckets") */
    int32_t fit_shard;     /* with slab_count > 1: 1 = this rank computes the local sets and
                              factors of its 1/slab_count share of the buckets only; the caller
                              all-gathers the blocks (lcp_fit_shard_buffers) and calls
                              lcp_fit_finish; 0 = every rank fits every bucket */
    double beta;           /* local_mode 1, 2: box enlargement in lengthscales (the paper uses 6) */
} lcp_opts_t;

/* per evaluated octree node (Alg. 1) */
typedef struct {
    int32_t level, i, j, k;   /* node index at `level` of the virtual 2^Lfull cube (R23) */
    int32_t ncase;            /* 0: M~ empty, 1: p1>a & p2>a, 2: p2<=a, 3: p1<=a (R8, R9) */
    int32_t refine;           /* subdivide (or emit, at max depth) */
    double p1, p2, U;         /* max P(Y_i<th), max P(Y_i>th) over M~ (-1 if empty), bound U */
} lcp_node_rec_t;

typedef struct {
    int64_t m;           /* observations */
    int32_t k;           /* local-GP size */
    int32_t nbuckets;
    int32_t nb[3];
    int32_t lfull;       /* depth of the full octree (2^lfull >= max cells) */
    int32_t bucket_side; /* cells per bucket side */
    int32_t device;
} lcp_info_t;

/* Create a context on CUDA device `device`.  `cuda_stream` is a cudaStream_t
 * (e.g. torch.cuda.current_stream().cuda_stream) or NULL for a private stream.
 * The ctx never destroys a caller-provided stream. */
lcp_status_t lcp_create(int32_t device, void* cuda_stream, lcp_ctx_t** out);
void lcp_destroy(lcp_ctx_t* ctx);
const char* lcp_last_error(const lcp_ctx_t* ctx);

/* a1-a4: bin the m observations into the bucket grid, gather each bucket's k
 * nearest observations (R2), build K_y = K_SS + nugget I, its Cholesky factor,
 * L^-1 and alpha = K_y^-1 (y_S - m0) per bucket (Eq. 1, PAPER.md:89-100;
 * local GP), and the observation marginals.
 *   xyz: m x 3 row-major, y: m; host pointers if on_device == 0 (copied inside,
 *   synchronously), else device pointers (read before return).
 *   opts may be NULL (bucket_log2 = 0, h_full = 2, FP64, one slab, automatic slab level, no records).
 * Errors: EINVAL (k < 1, k > m, variance <= 0, nugget < 0, lengthscale <= 0,
 * cells < 1, bucket_log2 > Lfull, a non-finite coordinate or value), EFACTOR,
 * ENUMERIC, ENOMEM, ECUDA. */
lcp_status_t lcp_fit_local(lcp_ctx_t* ctx, const double* xyz, const double* y, int64_t m,
                           int32_t on_device, const lcp_kernel_t* kernel, int32_t k,
                           const lcp_grid_t* grid, const lcp_opts_t* opts);

/* NEXT-2: the same as lcp_fit_local for a sparse-GP (SGPR) model: inducing
 * points xyz_M (m x 3), their posterior mean mu_M (m) and covariance A_M
 * (m x m row-major, symmetric, A_M <= K_MM) as stored after SGPR fitting
 * (PAPER.md:80-100).  Each bucket keeps its local inducing points (opts->local_mode:
 * its k nearest, or the beta-box set M' of PAPER.md:197-199) and evaluates Eq. 1
 * with the A_M term on them (whitened: v^T (I - L^-1 A L^-T) v, no
 * explicit K_SS^-1).  kernel->nugget is the jitter added to K_SS (e.g. 1e-9..1e-6
 * sigma_f^2).  Host or device pointers
 * as for lcp_fit_local.  Errors as lcp_fit_local, plus EINVAL for m > 60000 or a
 * non-finite A_M entry. */
lcp_status_t lcp_fit_sgpr(lcp_ctx_t* ctx, const double* xyz_M, const double* mu_M, const double* A_M,
                          int64_t m, int32_t on_device, const lcp_kernel_t* kernel, int32_t k,
                          const lcp_grid_t* grid, const lcp_opts_t* opts);

/* a5-a6: Alg. 1 as a level-synchronous pass over levels
 * 0..max_depth with the three-case preliminary test and the
 * Slepian bound U = 1 - B_l^d - B_u^d (Eq. 3-4; R6-R9).
 * Nodes with U <= threshold are pruned.  Returns the leaf cells (cells of
 * refined max-depth nodes) in a ctx-owned device array valid until the next
 * fit/refine/destroy.  Blocks the host (one size read-back per level).
 * With opts.brick_pass on (default when supported), the frontier of level
 * Lfull-2 -- aligned 4^3-cell bricks -- runs the brick pass: vertex marginals of
 * the bound lattice plus the isovalue-free 8-corner posterior and 8x8 factor of
 * every cell of the brick, kept until the next fit and reused by every later
 * lcp_pmc_cells* call whose cells they cover (any isovalue).
 * Errors: ESTATE before fit; EINVAL unless 0 < threshold < 0.5 and
 * 0 <= max_depth <= Lfull. */
lcp_status_t lcp_octree_refine(lcp_ctx_t* ctx, double isovalue, double threshold,
                               int32_t max_depth, int64_t* n_leaf_out,
                               const int64_t** leaf_cells_dev_out);

/* a7-a8: for each cell id, the 8-corner posterior of the cell's bucket local
 * GP, its 8x8 Cholesky (R14), and an N-sample Philox MC count
 * of samples whose corners straddle `isovalue` (R13, R13c, R24).
 *   cells: n_cells ids (device pointer if cells_on_device, else host);
 *   lcp_out: n_cells floats = count / n_samples (device pointer if
 *   out_on_device, else host: the call then synchronizes).
 * Any cell list is accepted (dense baseline = all ids).  Cells covered by the
 * brick-pass records of an earlier refine skip the posterior and factor; the
 * results are bit-identical either way.  Asynchronous on the ctx stream when
 * both pointers are device pointers (one 8-byte coverage read-back).
 * Errors: ESTATE; EINVAL (n_samples < 1 or > 2^31; a cell id outside
 * [0, nx*ny*nz): detected on the device before any kernel indexes by it and
 * reported by this call); ENUMERIC; ECUDA. */
lcp_status_t lcp_pmc_cells(lcp_ctx_t* ctx, const int64_t* cells, int64_t n_cells,
                           int32_t cells_on_device, double isovalue, int64_t n_samples,
                           uint64_t seed, uint32_t iso_index, float* lcp_out,
                           int32_t out_on_device);

/* a9: zero `field` (nx*ny*nz floats, device) and scatter lcp[q] into cell
 * cells[q] (every other cell is 0).  Asynchronous; an id outside
 * [0, nx*ny*nz) is skipped and reported as EINVAL by the next synchronizing call
 * (lcp_synchronize, or any call that blocks). */
lcp_status_t lcp_scatter_field(lcp_ctx_t* ctx, const int64_t* cells_dev, const float* lcp_dev,
                               int64_t n, float* field_dev);

/* One whole step of the path after fit: refine + pmc on the leaves + scatter
 * into the dense field (device pointer if out_on_device, else host, copied
 * before return).  n_leaf_out may be NULL. */
lcp_status_t lcp_run_field(lcp_ctx_t* ctx, double isovalue, double threshold, int32_t max_depth,
                           int64_t n_samples, uint64_t seed, uint32_t iso_index, float* field,
                           int32_t out_on_device, int64_t* n_leaf_out);

/* NEXT-3 fused multi-isovalue leaf pass (the paper's isovalue sweep,
 * PAPER.md:346, :386; reading R27).  For n_iso <= 16 isovalues: the 8-corner
 * posterior and its 8x8 Cholesky once per cell, and ONE Philox sample stream
 * per cell -- counter word 1 = `stream` (R13) -- whose every sample is tested
 * against each isovalue (ties cross).  Row t therefore equals
 * lcp_pmc_cells(cells, isovalues[t], ..., iso_index = stream) up to the FP32
 * rounding of y - isovalue (R25).
 *   cells_dev: n_cells ids; mask_dev: n_cells uint32 (bit t = cell is a leaf of
 *   isovalue t; a cleared bit writes 0), or NULL = all bits;
 *   lcp_dev: n_iso x n_cells floats, isovalue-major (caller-owned, device).
 * Asynchronous on the ctx stream.  Errors: ESTATE, EINVAL (n_iso not in
 * [1, 16], non-finite isovalue, n_samples < 1), ENUMERIC, ECUDA. */
lcp_status_t lcp_pmc_cells_multi(lcp_ctx_t* ctx, const int64_t* cells_dev, int64_t n_cells,
                                 const double* isovalues, int32_t n_iso, const uint32_t* mask_dev,
                                 int64_t n_samples, uint64_t seed, uint32_t stream, float* lcp_dev);

/* NEXT-3 whole step for n_iso <= 16 isovalues: Alg. 1 per isovalue (the vertex
 * marginal cache is shared), the union of the leaf sets in Morton order with a
 * per-cell isovalue mask, lcp_pmc_cells_multi on the union, and one dense field
 * per isovalue (0 off that isovalue's leaves).
 *   fields: n_iso x nx*ny*nz floats, isovalue-major (device pointer if
 *   out_on_device, else host, copied before return); n_leaf_out: n_iso leaf
 *   counts (may be NULL); n_union_out: union size (may be NULL).
 * Grids up to 2048 cells per axis.  Blocks the host.  Errors as
 * lcp_octree_refine and lcp_pmc_cells_multi. */
lcp_status_t lcp_run_field_multi(lcp_ctx_t* ctx, const double* isovalues, int32_t n_iso,
                                 double threshold, int32_t max_depth, int64_t n_samples,
                                 uint64_t seed, uint32_t stream, float* fields, int32_t out_on_device,
                                 int64_t* n_leaf_out, int64_t* n_union_out);

/* parity tap: the union leaf list (Morton order) and per-cell isovalue masks of
 * the last lcp_run_field_multi; ctx-owned device arrays. */
lcp_status_t lcp_union_cells(lcp_ctx_t* ctx, int64_t* n_out, const int64_t** cells_dev_out,
                             const uint32_t** mask_dev_out);

/* NEXT-4 level field: register a caller-owned device
 * array of nx*ny*nz bytes (NULL unregisters).  Every later refine writes, for
 * each cell, the octree level at which its region stopped: the level of the
 * pruned node containing it, or max_depth for leaf cells; 255 for cells outside
 * this rank's z-slab.  The array must stay valid while registered. */
lcp_status_t lcp_set_level_field(lcp_ctx_t* ctx, uint8_t* level_dev);

/* ---- parity taps (used by tests; not on the hot path) ---- */

/* node records of the last refine (opts.keep_records != 0), levels ascending,
 * Morton order within a level; ctx-owned device array. */
lcp_status_t lcp_node_records(lcp_ctx_t* ctx, int64_t* n_out, const lcp_node_rec_t** recs_dev_out);

/* FP64 posterior of cells (a7, as the leaf pass computes it): mu_dev n*8,
 * cov_dev n*64 (row-major 8x8), device.  Any list (duplicates allowed).
 * Errors: ESTATE, EINVAL (cell id out of range), ENUMERIC, ECUDA. */
lcp_status_t lcp_cell_posterior(lcp_ctx_t* ctx, const int64_t* cells_dev, int64_t n,
                                double* mu_dev, double* cov_dev);

/* local marginal (mean, variance before the floor) at points xyz_dev (n x 3),
 * using bucket bucket_dev[q] or, if bucket_dev == NULL, each point's own bucket.
 * Errors: ESTATE, EINVAL (a bucket id outside [0, nbuckets)), ENUMERIC, ECUDA. */
lcp_status_t lcp_point_marginals(lcp_ctx_t* ctx, const double* xyz_dev, int64_t n,
                                 const int32_t* bucket_dev, double* mu_dev, double* var_dev);

/* the local set of every bucket (nbuckets x k int32, ascending observation
 * indices; local_mode 1 pads a set smaller than k with -1), device */
lcp_status_t lcp_bucket_sets(lcp_ctx_t* ctx, int32_t* sets_dev);

lcp_status_t lcp_get_info(lcp_ctx_t* ctx, lcp_info_t* out);

/* JSON with per-phase device times and counters of the last calls */
lcp_status_t lcp_stats_json(lcp_ctx_t* ctx, char* buf, size_t cap);

/* wait for all work queued on the ctx stream; reports deferred device errors */
lcp_status_t lcp_synchronize(lcp_ctx_t* ctx);

/* Sharded fit (opts->fit_shard = 1, slab_count > 1): after lcp_fit_local /
 * lcp_fit_sgpr returned, the ctx holds the bucket blocks and local sets of its share
 * only.  Buckets are split by index: rank r owns [r per, (r+1) per) of the range padded
 * to slab_count x per.  bdata_dev / sets_dev (ctx-owned device arrays of slab_count x
 * chunk bytes; rank r's chunk at r x chunk) are to be all-gathered in place by the
 * caller (e.g. NCCL allgather with sendbuff = recvbuff + rank x chunk); then
 * lcp_fit_finish computes the observation marginals (a4) and completes the fit.
 * Every other call returns ESTATE in between.  The fitted model is the one an
 * unsharded fit builds, bit for bit (per-bucket arithmetic does not depend on the split).
 * Errors: EINVAL on a null pointer; ESTATE when no sharded fit is pending; lcp_fit_finish
 * as lcp_fit_local's a4 (ENUMERIC, ECUDA). */
lcp_status_t lcp_fit_shard_buffers(lcp_ctx_t* ctx, void** bdata_dev, int64_t* bdata_chunk_bytes,
                                   void** sets_dev, int64_t* sets_chunk_bytes);
lcp_status_t lcp_fit_finish(lcp_ctx_t* ctx);

/* ---- z-slab decomposition across GPUs (the paper itself is
 * single-process).  Host-only arithmetic, no device work, no ctx:
 * the rules lcp_octree_refine applies under opts.slab_count > 1, exposed so that
 * the caller can size and route the final gather (and test the plan on a CPU). */

/* automatic slab level for `slab_count` ranks on `grid` (opts.slab_level <= 0):
 * the shallowest level whose z-layers number >= 2 slab_count, at most
 * min(max_depth, Lfull - 3) and at least 1.  Returns -1 on bad arguments. */
int32_t lcp_slab_auto_level(const lcp_grid_t* grid, int32_t slab_count, int32_t max_depth);

/* contiguous z-layer ranges of `slab_count` ranks: cuts_out[0..slab_count]
 * (host, caller-owned), rank r owns layers [cuts_out[r], cuts_out[r+1]).  The cuts
 * minimise the largest rank weight (then the sum of squared rank weights; ties to
 * the earlier cut) over weights[0..n_layers) (host; >= 0; refine uses the expected
 * leaf work of the refined level-slab_level nodes of each layer: 1 + 1024 x the
 * fraction of their lattice vertices with both tails > threshold / 8); every rank
 * gets >= 1 layer when n_layers >= slab_count; all-zero weights give equal layer
 * counts.  LCP_EINVAL on null
 * pointers, n_layers < 1, slab_count < 1 or a negative weight. */
lcp_status_t lcp_slab_cuts(const int64_t* weights, int32_t n_layers, int32_t slab_count, int32_t* cuts_out);

#ifdef __cplusplus
}
#endif
#endif /* LCP_H */
