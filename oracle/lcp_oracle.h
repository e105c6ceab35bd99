/*
 * lcp_oracle.h -- plain FP64 CPU oracle for the LCP hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2512_12442_b200/) never links, imports or calls it, and
 * the two share no source, header, table or helper.
 *
 * Every function follows PAPER.md (arxiv 2512.12442) step by step; citations
 * are "PAPER.md:<line>" plus the equation / algorithm, readings "Rn" are listed
 * in DESIGN.md §2.  Compiled with -O2 -ffp-contract=off (no FMA contraction) so
 * the discrete decisions (bucket of a point, k-NN order) are reproducible.
 */
#ifndef LCP_ORACLE_H
#define LCP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t kind;          /* 0 = squared exponential, 1 = Matern-5/2 (BASELINE c4,c5) */
    int32_t pad_;
    double variance;       /* sigma_f^2 */
    double lengthscale[3]; /* per-axis l_d */
    double nugget;         /* observation noise variance sigma_n^2 (R1) */
    double prior_mean;     /* m0 */
} orc_kernel_t;

typedef struct {
    double lo[3], hi[3];
    int32_t cells[3];
    int32_t pad_;
} orc_grid_t;

typedef struct {
    int32_t level, i, j, k;   /* node (level, index) in the virtual 2^Lfull cube */
    int32_t ncase;            /* 0 empty M~, 1 both > alpha, 2 p2 <= alpha, 3 p1 <= alpha */
    int32_t refine;           /* U > alpha (or case 1) */
    double p1, p2, U;         /* p = -1 when M~ is empty */
} orc_node_rec_t;

typedef struct orc_model orc_model_t;

/* C1: kernel value. */
double orc_kernel(const orc_kernel_t* kern, const double* a, const double* b);

/* C2: exact GP joint posterior at nq query points (Eq. 1, with M = X).
 * mu: nq, cov: nq*nq row-major (may be NULL).  Returns 0, or 3 if K_y is not PD. */
int orc_gp_exact(const orc_kernel_t* kern, const double* X, const double* y, int64_t m,
                 const double* Q, int64_t nq, double* mu, double* cov);

/* C3-C4: bucket-local k-NN GP model (R2). */
int orc_model_create(const orc_kernel_t* kern, const orc_grid_t* grid, const double* X,
                     const double* y, int64_t m, int32_t k, int32_t bucket_log2,
                     int32_t h_full, orc_model_t** out);
void orc_model_destroy(orc_model_t* M);

/* R28 (NEXT-2): box mode -- bucket b's local set is every observation
 * inside the bucket box enlarged by beta l_d per axis (ascending index, at most k;
 * ORC_EINVAL if a box holds more than k, unless cap != 0: R28b, the |M'| cap -- such a
 * bucket takes its k nearest observations, R2, instead). */
int orc_model_create_box(const orc_kernel_t* kern, const orc_grid_t* grid, const double* X,
                         const double* y, int64_t m, int32_t k, int32_t bucket_log2,
                         int32_t h_full, double beta, int32_t cap, orc_model_t** out);
int32_t orc_model_nbuckets(const orc_model_t* M);
int32_t orc_model_lfull(const orc_model_t* M);
/* S_B of bucket b (ascending observation indices), k entries */
void orc_model_bucket_set(const orc_model_t* M, int32_t b, int32_t* idx_out);
int32_t orc_point_bucket(const orc_model_t* M, const double* x);
int32_t orc_vertex_bucket(const orc_model_t* M, int32_t i, int32_t j, int32_t k);
int32_t orc_cell_bucket(const orc_model_t* M, int64_t cell);

/* local GP marginal (mean, variance before floor) of the latent field at x, from bucket b */
int orc_local_marginal(const orc_model_t* M, int32_t b, const double* x, double* mu, double* var);

/* C8: 8-corner joint posterior of a cell (corner c = c0 + 2c1 + 4c2), from the cell's bucket.
 * mu: 8, cov: 64 row-major.  Returns 0 or 4 (variance < -1e-8 sigma_f^2). */
int orc_cell_posterior(const orc_model_t* M, int64_t cell, double* mu, double* cov);

/* C9: 8x8 Cholesky with PSD pivot clamp; L row-major 64 (upper part zero). */
void orc_chol8(const double* S, double* L);

/* C10: Philox4x32-10 block (Salmon et al. SC'11). ctr[4], key[2] -> out[4]. */
void orc_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out);

/* C10: the 8 standard normals of MC sample s of (cell, iso_index) under seed. */
void orc_normals8(uint64_t seed, int64_t cell, uint32_t iso_index, int64_t s, double* z);

/* C11: MC crossing count of one cell given mu[8] and L[64]. */
int64_t orc_mc_count(const double* mu, const double* L, double theta, int64_t n_samples,
                     uint64_t seed, int64_t cell, uint32_t iso_index);

/* Full leaf pass on a cell list: posterior, chol8, MC.  lcp_out[n] = count / N. */
int orc_pmc_cells(const orc_model_t* M, const int64_t* cells, int64_t n, double theta,
                  int64_t n_samples, uint64_t seed, uint32_t iso_index, double* lcp_out);

/* NEXT-3 (R27): fused multi-isovalue MC -- one sample stream (counter word 1 =
 * stream), the C11 crossing test for each of T thetas.  counts_out[T]. */
void orc_mc_count_multi(const double* mu, const double* L, const double* thetas, int32_t T,
                        int64_t n_samples, uint64_t seed, int64_t cell, uint32_t stream,
                        int64_t* counts_out);

/* NEXT-3: leaf pass for T <= 32 isovalues; mask[q] bit t (NULL = all) marks cell q
 * as a leaf of isovalue t (else LCP 0).  lcp_out[t * n + q]. */
int orc_pmc_cells_multi(const orc_model_t* M, const int64_t* cells, int64_t n, const double* thetas,
                        int32_t T, const uint32_t* mask, int64_t n_samples, uint64_t seed,
                        uint32_t stream, double* lcp_out);

/* C5: P(Y < theta), P(Y > theta) for Y ~ N(mu, var). */
void orc_tail_probs(double mu, double var, double theta, double* p_lo, double* p_hi);

/* NEXT-2: SGPR model (inducing points X_M, posterior mean mu_M, covariance A_M m x m
 * row-major): Eq. 1 globally, and restricted to each bucket's k
 * nearest inducing points.  kern->nugget is the jitter added to K_MM. */
int orc_sgpr_exact(const orc_kernel_t* kern, const double* XM, const double* muM, const double* AM, int64_t m,
                   const double* Q, int64_t nq, double* mu, double* cov);
int orc_model_create_sgpr(const orc_kernel_t* kern, const orc_grid_t* grid, const double* XM, const double* muM,
                          const double* AM, int64_t m, int32_t k, int32_t bucket_log2, int32_t h_full,
                          orc_model_t** out);
/* the same with the local sets of local_mode 0 (k-NN), 1 (beta-box) or 2 (capped beta-box) */
int orc_model_create_sgpr_mode(const orc_kernel_t* kern, const orc_grid_t* grid, const double* XM,
                               const double* muM, const double* AM, int64_t m, int32_t k, int32_t bucket_log2,
                               int32_t h_full, int32_t local_mode, double beta, orc_model_t** out);

/* NEXT-1 (R26): continuous extreme search at nodes with h > h_full; iters = 0 disables. */
void orc_model_set_extreme(orc_model_t* M, int32_t iters);
/* f = (mu - theta) / (sigma sqrt 2) of bucket b's local GP at x, and grad f (3) */
double orc_local_f_grad(const orc_model_t* M, int32_t b, const double* x, double theta, double* grad);

/* test tap: {lattice zmax, lattice zmin, searched zmax, searched zmin} of a node (R26) */
void orc_node_extremes(const orc_model_t* M, double theta, int32_t level, int32_t i, int32_t j, int32_t k,
                       double* out);

/* C6: evaluate one octree node (Alg. 1 lines 2-13, Eq. 3-4). */
int orc_eval_node(const orc_model_t* M, double theta, double alpha, int32_t level,
                  int32_t i, int32_t j, int32_t k, orc_node_rec_t* rec);

/* C7: level-synchronous octree (Alg. 1), restricted to the subtree of
 * (sub_level, si, sj, sk) when sub_level >= 0 (the levels above are not recorded).
 * Records every evaluated node; leaves are the cells of refined depth-D nodes,
 * returned sorted ascending.  Outputs are malloc'ed; free with orc_free. */
int orc_octree(const orc_model_t* M, double theta, double alpha, int32_t max_depth,
               int32_t sub_level, int32_t si, int32_t sj, int32_t sk,
               orc_node_rec_t** recs, int64_t* n_recs, int64_t** leaves, int64_t* n_leaves);
void orc_free(void* p);

int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
