/*
 * lcp_oracle.c -- plain, slow, obviously correct FP64 CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY (see lcp_oracle.h).  Shares no code with the CUDA
 * path.  Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC.
 *
 * Conventions (C0): cell size h_d = (hi_d - lo_d) / cells_d;
 * vertex (i,j,k) sits at lo + (i,j,k) h; cell id = i + nx (j + ny k);
 * corner c = c0 + 2 c1 + 4 c2 is vertex (i+c0, j+c1, k+c2);
 * the octree lives on a virtual cube of 2^Lfull cells per axis anchored at lo.
 *
 * Parallelism: only `#pragma omp parallel for` over independent buckets,
 * nodes or cells; every per-item computation is the sequential definition.
 */
#include "lcp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_EFACTOR 3
#define ORC_ENUMERIC 4

static const double ORC_SQRT2 = 1.4142135623730951;
static const double ORC_PI = 3.141592653589793;

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_free(void* p) { free(p); }

/* ------------------------------------------------------------------ C1 --- */
/* SE: sigma^2 exp(-|x1-x2|^2 / (2 l^2)), per-axis l (BASELINE c3).
 * Matern-5/2 (BASELINE c4, c5): r = |(x1-x2)/l|, sigma^2 (1 + sqrt5 r + 5/3 r^2) e^{-sqrt5 r}. */
double orc_kernel(const orc_kernel_t* kern, const double* a, const double* b) {
    double r2 = 0.0;
    for (int d = 0; d < 3; ++d) {
        double t = (a[d] - b[d]) / kern->lengthscale[d];
        r2 += t * t;
    }
    if (kern->kind == 0) return kern->variance * exp(-0.5 * r2);
    double r = sqrt(r2);
    double s5 = sqrt(5.0);
    return kern->variance * (1.0 + s5 * r + (5.0 / 3.0) * r2) * exp(-s5 * r);
}

/* ------------------------------------------------------ dense helpers --- */
/* Cholesky A = L L^T of an n x n row-major SPD matrix (lower written into L). */
static int chol_plain(const double* A, double* L, int n) {
    memset(L, 0, sizeof(double) * (size_t)n * n);
    for (int j = 0; j < n; ++j) {
        double s = A[(size_t)j * n + j];
        for (int p = 0; p < j; ++p) s -= L[(size_t)j * n + p] * L[(size_t)j * n + p];
        if (!(s > 0.0)) return ORC_EFACTOR;
        double ljj = sqrt(s);
        L[(size_t)j * n + j] = ljj;
        for (int i = j + 1; i < n; ++i) {
            double t = A[(size_t)i * n + j];
            for (int p = 0; p < j; ++p) t -= L[(size_t)i * n + p] * L[(size_t)j * n + p];
            L[(size_t)i * n + j] = t / ljj;
        }
    }
    return ORC_OK;
}

/* K_y = K + sigma_n^2 I; on failure retry with jitter 1e-10, 1e-9, 1e-8 x sigma_f^2 (R15). */
static int chol_jitter(double* A, double* L, int n, double variance) {
    if (chol_plain(A, L, n) == ORC_OK) return ORC_OK;
    double jit = 1e-10 * variance, added = 0.0;
    for (int t = 0; t < 3; ++t, jit *= 10.0) {
        for (int i = 0; i < n; ++i) A[(size_t)i * n + i] += jit - added;
        added = jit;
        if (chol_plain(A, L, n) == ORC_OK) return ORC_OK;
    }
    return ORC_EFACTOR;
}

/* forward substitution L v = b */
static void forward_sub(const double* L, int n, const double* b, double* v) {
    for (int i = 0; i < n; ++i) {
        double t = b[i];
        for (int p = 0; p < i; ++p) t -= L[(size_t)i * n + p] * v[p];
        v[i] = t / L[(size_t)i * n + i];
    }
}

/* backward substitution L^T v = b */
static void backward_sub(const double* L, int n, const double* b, double* v) {
    for (int i = n - 1; i >= 0; --i) {
        double t = b[i];
        for (int p = i + 1; p < n; ++p) t -= L[(size_t)p * n + i] * v[p];
        v[i] = t / L[(size_t)i * n + i];
    }
}

/* ------------------------------------------------------------------ C2 --- */
/* Exact GP regression posterior = Eq. 1 with M = X,
 * mu_M = K (K + s_n^2 I)^-1 y, A_M = s_n^2 K (K + s_n^2 I)^-1 (R1):
 *   mu(I)    = m0 + K_IX alpha,            alpha = K_y^-1 (y - m0)
 *   Sigma(I) = K_II - V^T V,               V = L^-1 K_XI,  K_y = L L^T          */
int orc_gp_exact(const orc_kernel_t* kern, const double* X, const double* y, int64_t m,
                 const double* Q, int64_t nq, double* mu, double* cov) {
    int n = (int)m;
    double* A = malloc(sizeof(double) * n * n);
    double* L = malloc(sizeof(double) * n * n);
    double* r = malloc(sizeof(double) * n);
    double* w = malloc(sizeof(double) * n);
    double* alpha = malloc(sizeof(double) * n);
    double* V = malloc(sizeof(double) * n * (nq > 0 ? nq : 1));
    double* kq = malloc(sizeof(double) * n);
    int st = ORC_OK;
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b)
            A[a * n + b] = orc_kernel(kern, X + 3 * a, X + 3 * b) + (a == b ? kern->nugget : 0.0);
    st = chol_jitter(A, L, n, kern->variance);
    if (st == ORC_OK) {
        for (int a = 0; a < n; ++a) r[a] = y[a] - kern->prior_mean;
        forward_sub(L, n, r, w);
        backward_sub(L, n, w, alpha);
        for (int64_t q = 0; q < nq; ++q) {
            double s = 0.0;
            for (int a = 0; a < n; ++a) {
                kq[a] = orc_kernel(kern, X + 3 * a, Q + 3 * q);
                s += kq[a] * alpha[a];
            }
            mu[q] = kern->prior_mean + s;
            forward_sub(L, n, kq, V + (size_t)q * n);
        }
        if (cov) {
            for (int64_t p = 0; p < nq; ++p)
                for (int64_t q = 0; q < nq; ++q) {
                    double s = orc_kernel(kern, Q + 3 * p, Q + 3 * q);
                    for (int a = 0; a < n; ++a) s -= V[(size_t)p * n + a] * V[(size_t)q * n + a];
                    cov[p * nq + q] = s;
                }
        }
    }
    free(A); free(L); free(r); free(w); free(alpha); free(V); free(kq);
    return st;
}

/* --------------------------------------------------------------- C3-C4 --- */
struct orc_model {
    orc_kernel_t kern;
    orc_grid_t grid;
    double h[3];          /* cell size */
    double w[3];          /* k-NN metric weights 1 / l_d */
    int32_t lfull, b, bs, h_full;
    int32_t extreme_iters;  /* NEXT-1: projected-gradient iterations at nodes with h > h_full (0 = off) */
    int32_t nb[3], nbuckets;
    int32_t m, k;
    double* X;            /* m x 3 */
    double* y;            /* m */
    int32_t* S;           /* nbuckets x k, ascending observation index (box mode: kb[b] used, -1 after) */
    int32_t* kb;          /* box mode (R28): per-bucket set size <= k; NULL = k-NN mode (every set has k) */
    double beta;          /* box mode: enlargement of the bucket box in units of l_d */
    double* L;            /* nbuckets x k x k, lower factor of K_y(S_B) */
    double* alpha;        /* nbuckets x k */
    double* B;            /* NEXT-2 SGPR mode: nbuckets x k x k, B = L^-1 A_SS L^-T (stride = set size; NULL: GP
                             regression); Eq. 1's third term K_xS W A_SS W K_Sx = v^T B v with v = L^-1 K_Sx */
    int32_t cap;          /* box mode, R28b: a bucket whose box holds > k observations takes its k-NN set */
    double* mu_obs;       /* m: local marginal at x_i from bucket(x_i) (R10) */
    double* var_obs;      /* m (floored) */
    int32_t* obs_cell;    /* m x 3 finest cell of x_i (clamped) */
};

static int32_t clampi(int64_t v, int32_t lo, int32_t hi) {
    return (int32_t)(v < lo ? lo : (v > hi ? hi : v));
}

int32_t orc_model_nbuckets(const orc_model_t* M) { return M->nbuckets; }
int32_t orc_model_lfull(const orc_model_t* M) { return M->lfull; }

/* R3: point -> bucket floor((x - lo) / s_B) clamped, s_B = bs * h. */
int32_t orc_point_bucket(const orc_model_t* M, const double* x) {
    int32_t idx[3];
    for (int d = 0; d < 3; ++d) {
        double sB = (double)M->bs * M->h[d];
        double t = floor((x[d] - M->grid.lo[d]) / sB);
        idx[d] = clampi((int64_t)(t < -1.0 ? -1.0 : (t > 2e9 ? 2e9 : t)), 0, M->nb[d] - 1);
    }
    return idx[0] + M->nb[0] * (idx[1] + M->nb[1] * idx[2]);
}

/* R3: vertex (i,j,k) -> bucket min(i / bs, nb - 1) per axis. */
int32_t orc_vertex_bucket(const orc_model_t* M, int32_t i, int32_t j, int32_t k) {
    int32_t v[3] = {i, j, k}, idx[3];
    for (int d = 0; d < 3; ++d) idx[d] = clampi(v[d] / M->bs, 0, M->nb[d] - 1);
    return idx[0] + M->nb[0] * (idx[1] + M->nb[1] * idx[2]);
}

/* R3: cell -> bucket containing it (bucket boundaries are cell boundaries). */
int32_t orc_cell_bucket(const orc_model_t* M, int64_t cell) {
    int64_t nx = M->grid.cells[0], ny = M->grid.cells[1];
    int32_t i = (int32_t)(cell % nx), j = (int32_t)((cell / nx) % ny), k = (int32_t)(cell / (nx * ny));
    return orc_vertex_bucket(M, i, j, k);
}

/* size of bucket b's local set (k in k-NN mode) */
static int set_size(const orc_model_t* M, int32_t b) { return M->kb ? M->kb[b] : M->k; }

void orc_model_bucket_set(const orc_model_t* M, int32_t b, int32_t* idx_out) {
    int kb = set_size(M, b);
    memcpy(idx_out, M->S + (size_t)b * M->k, sizeof(int32_t) * kb);
    for (int a = kb; a < M->k; ++a) idx_out[a] = -1;
}

typedef struct { double d2; int32_t idx; } knn_item;

static int knn_cmp(const void* pa, const void* pb) {
    const knn_item* a = pa; const knn_item* b = pb;
    if (a->d2 < b->d2) return -1;
    if (a->d2 > b->d2) return 1;
    return (a->idx > b->idx) - (a->idx < b->idx);
}

static int int_cmp(const void* pa, const void* pb) {
    int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
    return (a > b) - (a < b);
}

static void vertex_pos(const orc_model_t* M, int32_t i, int32_t j, int32_t k, double* x) {
    x[0] = M->grid.lo[0] + (double)i * M->h[0];
    x[1] = M->grid.lo[1] + (double)j * M->h[1];
    x[2] = M->grid.lo[2] + (double)k * M->h[2];
}

int orc_local_marginal(const orc_model_t* M, int32_t b, const double* x, double* mu, double* var) {
    int ks = M->k, k = set_size(M, b);
    const int32_t* S = M->S + (size_t)b * ks;
    const double* L = M->L + (size_t)b * ks * ks;   /* k x k, stride k */
    const double* al = M->alpha + (size_t)b * ks;
    double* kv = malloc(sizeof(double) * k);
    double* v = malloc(sizeof(double) * k);
    double s = 0.0;
    for (int a = 0; a < k; ++a) {
        kv[a] = orc_kernel(&M->kern, M->X + 3 * (size_t)S[a], x);
        s += kv[a] * al[a];
    }
    *mu = M->kern.prior_mean + s;
    forward_sub(L, k, kv, v);
    double q = orc_kernel(&M->kern, x, x);
    for (int a = 0; a < k; ++a) q -= v[a] * v[a];
    if (M->B) {   /* + K_xS W A_SS W K_Sx = v^T B v (Eq. 1, third term; W = L^-T L^-1) */
        const double* Bb = M->B + (size_t)b * ks * ks;
        for (int a = 0; a < k; ++a)
            for (int c = 0; c < k; ++c) q += v[a] * Bb[(size_t)a * k + c] * v[c];
    }
    *var = q;
    free(kv); free(v);
    return ORC_OK;
}

/* R16: variance floor 1e-12 sigma_f^2, error below -1e-8 sigma_f^2. */
static int floor_var(const orc_model_t* M, double var, double* out) {
    if (var < -1e-8 * M->kern.variance) return ORC_ENUMERIC;
    double f = 1e-12 * M->kern.variance;
    *out = var > f ? var : f;
    return ORC_OK;
}

/* R28 box mode: bucket b's local set is every observation in the bucket box enlarged
 * by beta l_d per axis, [lo_b - beta l, hi_b + beta l) (the paper's
 * beta-l box with beta = 6 at P:423), ascending index; EINVAL if a set exceeds k.
 * Bounds evaluated left to right without FMA (bit-identical to the GPU's). */
static int box_set(const orc_model_t* M, int32_t bkt, const double* X, int64_t m, int32_t* S, int32_t k) {
    int32_t bi[3] = {bkt % M->nb[0], (bkt / M->nb[0]) % M->nb[1], bkt / (M->nb[0] * M->nb[1])};
    double lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
        double w = M->beta * M->kern.lengthscale[d];
        lo[d] = (M->grid.lo[d] + (double)(bi[d] * M->bs) * M->h[d]) - w;
        hi[d] = (M->grid.lo[d] + (double)((bi[d] + 1) * M->bs) * M->h[d]) + w;
    }
    int n = 0;
    for (int64_t i = 0; i < m; ++i) {
        int in = 1;
        for (int d = 0; d < 3; ++d) in = in && X[3 * i + d] >= lo[d] && X[3 * i + d] < hi[d];
        if (in) {
            if (n >= k) return -1;
            S[n++] = (int32_t)i;
        }
    }
    return n;
}

static int model_create(const orc_kernel_t* kern, const orc_grid_t* grid, const double* X,
                        const double* y, int64_t m, int32_t k, int32_t bucket_log2,
                        int32_t h_full, double beta, int32_t cap, orc_model_t** out);

int orc_model_create(const orc_kernel_t* kern, const orc_grid_t* grid, const double* X,
                     const double* y, int64_t m, int32_t k, int32_t bucket_log2,
                     int32_t h_full, orc_model_t** out) {
    return model_create(kern, grid, X, y, m, k, bucket_log2, h_full, 0.0, 0, out);
}

int orc_model_create_box(const orc_kernel_t* kern, const orc_grid_t* grid, const double* X,
                         const double* y, int64_t m, int32_t k, int32_t bucket_log2,
                         int32_t h_full, double beta, int32_t cap, orc_model_t** out) {
    if (!(beta > 0.0)) return ORC_EINVAL;
    return model_create(kern, grid, X, y, m, k, bucket_log2, h_full, beta, cap, out);
}

static int model_create(const orc_kernel_t* kern, const orc_grid_t* grid, const double* X,
                        const double* y, int64_t m, int32_t k, int32_t bucket_log2,
                        int32_t h_full, double beta, int32_t cap, orc_model_t** out) {
    *out = NULL;
    if (m < 1 || k < 1 || k > m || bucket_log2 < 0 || h_full < 0) return ORC_EINVAL;
    if (kern->variance <= 0 || kern->nugget < 0) return ORC_EINVAL;
    for (int d = 0; d < 3; ++d)
        if (grid->cells[d] < 1 || !(grid->hi[d] > grid->lo[d]) || kern->lengthscale[d] <= 0)
            return ORC_EINVAL;
    orc_model_t* M = calloc(1, sizeof(orc_model_t));
    M->kern = *kern;
    M->grid = *grid;
    int32_t cmax = grid->cells[0];
    if (grid->cells[1] > cmax) cmax = grid->cells[1];
    if (grid->cells[2] > cmax) cmax = grid->cells[2];
    int32_t lf = 0;
    while ((1 << lf) < cmax) ++lf;
    M->lfull = lf;
    if (bucket_log2 > lf) { free(M); return ORC_EINVAL; }
    M->b = bucket_log2;
    M->bs = 1 << (lf - bucket_log2);
    M->h_full = h_full;
    for (int d = 0; d < 3; ++d) {
        M->h[d] = (grid->hi[d] - grid->lo[d]) / (double)grid->cells[d];
        M->w[d] = 1.0 / kern->lengthscale[d];
        M->nb[d] = (grid->cells[d] + M->bs - 1) / M->bs;
    }
    M->nbuckets = M->nb[0] * M->nb[1] * M->nb[2];
    M->m = (int32_t)m;
    M->k = k;
    M->beta = beta;
    M->cap = cap;
    if (beta > 0.0) M->kb = malloc(sizeof(int32_t) * (size_t)M->nbuckets);
    M->X = malloc(sizeof(double) * 3 * m);
    M->y = malloc(sizeof(double) * m);
    memcpy(M->X, X, sizeof(double) * 3 * m);
    memcpy(M->y, y, sizeof(double) * m);
    M->S = malloc(sizeof(int32_t) * (size_t)M->nbuckets * k);
    M->L = malloc(sizeof(double) * (size_t)M->nbuckets * k * k);
    M->alpha = malloc(sizeof(double) * (size_t)M->nbuckets * k);
    int status = ORC_OK;

#pragma omp parallel for schedule(dynamic)
    for (int32_t bkt = 0; bkt < M->nbuckets; ++bkt) {
        int32_t bi[3] = {bkt % M->nb[0], (bkt / M->nb[0]) % M->nb[1], bkt / (M->nb[0] * M->nb[1])};
        double c[3];
        for (int d = 0; d < 3; ++d) c[d] = grid->lo[d] + ((double)bi[d] + 0.5) * ((double)M->bs * M->h[d]);
        int32_t* S = M->S + (size_t)bkt * k;
        int kb = k;
        int use_knn = beta <= 0.0;
        if (beta > 0.0) {
            kb = box_set(M, bkt, X, m, S, k);
            if (kb < 0 && M->cap) {          /* R28b: the |M'| cap -- this bucket takes its k-NN set */
                use_knn = 1;
                kb = k;
            } else if (kb < 0) {
#pragma omp critical
                status = ORC_EINVAL;
                kb = 0;
            }
            M->kb[bkt] = kb;
            if (!use_knn)
                for (int a = kb; a < k; ++a) S[a] = -1;
        }
        if (use_knn) {
            /* k nearest in the metric sum_d ((x_d - c_d) w_d)^2, ties -> lower index (R2) */
            knn_item* it = malloc(sizeof(knn_item) * m);
            for (int64_t i = 0; i < m; ++i) {
                double t0 = (X[3 * i + 0] - c[0]) * M->w[0];
                double t1 = (X[3 * i + 1] - c[1]) * M->w[1];
                double t2 = (X[3 * i + 2] - c[2]) * M->w[2];
                it[i].d2 = t0 * t0 + t1 * t1 + t2 * t2;
                it[i].idx = (int32_t)i;
            }
            qsort(it, m, sizeof(knn_item), knn_cmp);
            for (int a = 0; a < k; ++a) S[a] = it[a].idx;
            qsort(S, k, sizeof(int32_t), int_cmp);
            free(it);
        }
        /* K_y = K(S,S) + sigma_n^2 I; L = chol(K_y); alpha = K_y^-1 (y_S - m0)  (Eq. 1, R1);
         * box mode: the kb x kb system of the bucket's set (L stored with stride kb) */
        const int kk = kb;
        double* A = malloc(sizeof(double) * (kk > 0 ? kk * kk : 1));
        double* Lb = M->L + (size_t)bkt * k * k;
        for (int a = 0; a < kk; ++a)
            for (int b2 = 0; b2 < kk; ++b2)
                A[a * kk + b2] = orc_kernel(kern, X + 3 * (size_t)S[a], X + 3 * (size_t)S[b2]) +
                                 (a == b2 ? kern->nugget : 0.0);
        int st = kk > 0 ? chol_jitter(A, Lb, kk, kern->variance) : ORC_OK;
        if (st != ORC_OK) {
#pragma omp critical
            status = st;
        } else {
            double* r = malloc(sizeof(double) * (kk > 0 ? kk : 1));
            double* w = malloc(sizeof(double) * (kk > 0 ? kk : 1));
            for (int a = 0; a < kk; ++a) r[a] = y[S[a]] - kern->prior_mean;
            forward_sub(Lb, kk, r, w);
            backward_sub(Lb, kk, w, M->alpha + (size_t)bkt * k);
            free(r); free(w);
        }
        free(A);
    }
    if (status != ORC_OK) { orc_model_destroy(M); return status; }

    /* a4: observation marginals and finest cells (R10) */
    M->mu_obs = malloc(sizeof(double) * m);
    M->var_obs = malloc(sizeof(double) * m);
    M->obs_cell = malloc(sizeof(int32_t) * 3 * m);
    for (int64_t i = 0; i < m; ++i) {
        double var;
        orc_local_marginal(M, orc_point_bucket(M, X + 3 * i), X + 3 * i, &M->mu_obs[i], &var);
        if (floor_var(M, var, &M->var_obs[i]) != ORC_OK) status = ORC_ENUMERIC;
        for (int d = 0; d < 3; ++d) {
            double t = floor((X[3 * i + d] - grid->lo[d]) / M->h[d]);
            M->obs_cell[3 * i + d] = clampi((int64_t)(t < -1.0 ? -1.0 : (t > 2e9 ? 2e9 : t)), 0, grid->cells[d] - 1);
        }
    }
    if (status != ORC_OK) { orc_model_destroy(M); return status; }
    *out = M;
    return ORC_OK;
}

void orc_model_destroy(orc_model_t* M) {
    if (!M) return;
    free(M->X); free(M->y); free(M->S); free(M->kb); free(M->L); free(M->alpha); free(M->B);
    free(M->mu_obs); free(M->var_obs); free(M->obs_cell);
    free(M);
}

/* ---------------------------------------------------------------- NEXT-2 --- */
/* B = L^-1 A L^-T for the Cholesky factor L of K_MM (n x n, A row-major with row
 * stride lda, rows/cols indexed through idx, or the identity map if idx == NULL):
 * column c of T = L^-1 A by forward substitution, then row r of B solves L x = T[r, :]^T.
 * With W = K_MM^-1 = L^-T L^-1, K_IM W A W K_MI = v^T B v for v = L^-1 K_MI. */
static void whiten_A(const double* L, int n, const double* A, int64_t lda, const int32_t* idx, double* B) {
    double* col = malloc(sizeof(double) * n);
    double* t = malloc(sizeof(double) * n);
    double* T = malloc(sizeof(double) * (size_t)n * n);
    for (int c = 0; c < n; ++c) {
        for (int r = 0; r < n; ++r) {
            int64_t ir = idx ? idx[r] : r, ic = idx ? idx[c] : c;
            col[r] = A[(size_t)ir * lda + ic];
        }
        forward_sub(L, n, col, t);
        for (int r = 0; r < n; ++r) T[(size_t)r * n + c] = t[r];
    }
    for (int r = 0; r < n; ++r) {
        forward_sub(L, n, T + (size_t)r * n, t);
        for (int c = 0; c < n; ++c) B[(size_t)r * n + c] = t[c];
    }
    free(col); free(t); free(T);
}

/* Eq. 1 for an SGPR model (inducing points X_M, their posterior mean
 * mu_M and covariance A_M, m x m row-major):
 *   mu_I    = m0 + K_IM K_MM^-1 (mu_M - m0)
 *   Sigma_I = K_II - K_IM K_MM^-1 K_MI + K_IM K_MM^-1 A_M K_MM^-1 K_MI,
 * with K_MM + jitter I (jitter = kern->nugget) = L L^T.  K_MM^-1 = L^-T L^-1 is applied
 * by triangular solves: v = L^-1 K_MI, the second term is v^T v and the third v^T B v
 * with B = L^-1 A_M L^-T (no explicit inverse: the product with an explicit K_MM^-1
 * loses ~cond(K_MM) eps, 4e-7 sigma_f^2 on ill-conditioned SGPR fits, against ~1e-9
 * here; tests/test_oracle_sgpr.py pins this against extended precision). */
int orc_sgpr_exact(const orc_kernel_t* kern, const double* XM, const double* muM, const double* AM, int64_t m,
                   const double* Q, int64_t nq, double* mu, double* cov) {
    int n = (int)m;
    double* K = malloc(sizeof(double) * n * n);
    double* L = malloc(sizeof(double) * n * n);
    double* B = malloc(sizeof(double) * n * n);
    double* V = malloc(sizeof(double) * nq * n);   /* v_q = L^-1 K_Mq */
    double* kq = malloc(sizeof(double) * n);
    double* r = malloc(sizeof(double) * n);
    double* w = malloc(sizeof(double) * n);
    double* al = malloc(sizeof(double) * n);
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b)
            K[a * n + b] = orc_kernel(kern, XM + 3 * a, XM + 3 * b) + (a == b ? kern->nugget : 0.0);
    int st = chol_jitter(K, L, n, kern->variance);
    if (st == ORC_OK) {
        for (int a = 0; a < n; ++a) r[a] = muM[a] - kern->prior_mean;
        forward_sub(L, n, r, w);                  /* alpha = K_MM^-1 (mu_M - m0) */
        backward_sub(L, n, w, al);
        whiten_A(L, n, AM, m, NULL, B);
        for (int64_t q = 0; q < nq; ++q) {
            double s = 0.0;
            for (int a = 0; a < n; ++a) {
                kq[a] = orc_kernel(kern, Q + 3 * q, XM + 3 * a);
                s += kq[a] * al[a];
            }
            mu[q] = kern->prior_mean + s;
            forward_sub(L, n, kq, V + (size_t)q * n);
        }
        if (cov)
            for (int64_t p = 0; p < nq; ++p)
                for (int64_t q = 0; q < nq; ++q) {
                    const double* vp = V + (size_t)p * n;
                    const double* vq = V + (size_t)q * n;
                    double s = orc_kernel(kern, Q + 3 * p, Q + 3 * q);
                    for (int a = 0; a < n; ++a) s -= vp[a] * vq[a];
                    for (int a = 0; a < n; ++a)
                        for (int b = 0; b < n; ++b) s += vp[a] * B[(size_t)a * n + b] * vq[b];
                    cov[p * nq + q] = s;
                }
    }
    free(K); free(L); free(B); free(V); free(kq); free(r); free(w); free(al);
    return st;
}

/* Bucket-local SGPR: each bucket keeps its local inducing points S -- the k nearest
 * (R2), or the beta-box set (R28; local_mode 2: capped at k by R28b) -- and Eq. 1
 * restricted to S: L = chol(K_SS + jitter), alpha = K_SS^-1 (mu_S - m0) by solves,
 * B = L^-1 A_SS L^-T.  Marginals / cell posteriors add the third term v^T B v. */
int orc_model_create_sgpr_mode(const orc_kernel_t* kern, const orc_grid_t* grid, const double* XM,
                               const double* muM, const double* AM, int64_t m, int32_t k, int32_t bucket_log2,
                               int32_t h_full, int32_t local_mode, double beta, orc_model_t** out) {
    /* the local sets, K_SS factor and alpha are the GP-regression model with nugget = jitter */
    int st = local_mode == 0 ? orc_model_create(kern, grid, XM, muM, m, k, bucket_log2, h_full, out)
                             : orc_model_create_box(kern, grid, XM, muM, m, k, bucket_log2, h_full, beta,
                                                    local_mode == 2, out);
    if (st != ORC_OK) return st;
    orc_model_t* M = *out;
    M->B = calloc((size_t)M->nbuckets * k * k, sizeof(double));
#pragma omp parallel for schedule(dynamic)
    for (int32_t bkt = 0; bkt < M->nbuckets; ++bkt) {
        const int kb = set_size(M, bkt);
        if (kb > 0)
            whiten_A(M->L + (size_t)bkt * k * k, kb, AM, m, M->S + (size_t)bkt * k, M->B + (size_t)bkt * k * k);
    }
    /* observation marginals now include the A term */
    for (int64_t i = 0; i < m; ++i) {
        double var;
        orc_local_marginal(M, orc_point_bucket(M, XM + 3 * i), XM + 3 * i, &M->mu_obs[i], &var);
        if (floor_var(M, var, &M->var_obs[i]) != ORC_OK) { orc_model_destroy(M); *out = NULL; return ORC_ENUMERIC; }
    }
    return ORC_OK;
}

int orc_model_create_sgpr(const orc_kernel_t* kern, const orc_grid_t* grid, const double* XM, const double* muM,
                          const double* AM, int64_t m, int32_t k, int32_t bucket_log2, int32_t h_full,
                          orc_model_t** out) {
    return orc_model_create_sgpr_mode(kern, grid, XM, muM, AM, m, k, bucket_log2, h_full, 0, 0.0, out);
}

/* ------------------------------------------------------------------ C8 --- */
int orc_cell_posterior(const orc_model_t* M, int64_t cell, double* mu, double* cov) {
    int64_t nx = M->grid.cells[0], ny = M->grid.cells[1];
    int32_t ci = (int32_t)(cell % nx), cj = (int32_t)((cell / nx) % ny), ck = (int32_t)(cell / (nx * ny));
    int32_t b = orc_vertex_bucket(M, ci, cj, ck);
    int ks = M->k, k = set_size(M, b);
    const int32_t* S = M->S + (size_t)b * ks;
    const double* L = M->L + (size_t)b * ks * ks;
    const double* al = M->alpha + (size_t)b * ks;
    double xc[8][3];
    for (int c = 0; c < 8; ++c) vertex_pos(M, ci + (c & 1), cj + ((c >> 1) & 1), ck + (c >> 2), xc[c]);
    double* K = malloc(sizeof(double) * 8 * k);
    double* V = malloc(sizeof(double) * 8 * k);
    for (int c = 0; c < 8; ++c) {
        double s = 0.0;
        double* Kc = K + (size_t)c * k;
        for (int a = 0; a < k; ++a) {
            Kc[a] = orc_kernel(&M->kern, M->X + 3 * (size_t)S[a], xc[c]);
            s += Kc[a] * al[a];
        }
        mu[c] = M->kern.prior_mean + s;
        forward_sub(L, k, Kc, V + (size_t)c * k);
    }
    int st = ORC_OK;
    const double* Bb = M->B ? M->B + (size_t)b * ks * ks : NULL;
    for (int c = 0; c < 8; ++c)
        for (int e = 0; e < 8; ++e) {
            double s = orc_kernel(&M->kern, xc[c], xc[e]);
            for (int a = 0; a < k; ++a) s -= V[(size_t)c * k + a] * V[(size_t)e * k + a];
            if (Bb)   /* + K_cS W A_SS W K_Se = v_c^T B v_e (Eq. 1, third term) */
                for (int a = 0; a < k; ++a)
                    for (int d = 0; d < k; ++d) s += V[(size_t)c * k + a] * Bb[(size_t)a * k + d] * V[(size_t)e * k + d];
            cov[c * 8 + e] = s;
        }
    for (int c = 0; c < 8; ++c)
        if (cov[c * 8 + c] < -1e-8 * M->kern.variance) st = ORC_ENUMERIC;
    free(K); free(V);
    return st;
}

/* ------------------------------------------------------------------ C9 --- */
/* Cholesky of the 8x8 corner covariance; a pivot <= 1e-12 max_diag is clamped:
 * L_jj = 0 and the column below is zeroed (PSD clamp, never fails; R14). */
void orc_chol8(const double* S, double* L) {
    double md = 0.0;
    for (int c = 0; c < 8; ++c) if (S[c * 8 + c] > md) md = S[c * 8 + c];
    double tol = 1e-12 * md;
    memset(L, 0, sizeof(double) * 64);
    for (int j = 0; j < 8; ++j) {
        double s = S[j * 8 + j];
        for (int p = 0; p < j; ++p) s -= L[j * 8 + p] * L[j * 8 + p];
        if (s <= tol) continue;  /* column stays zero */
        double ljj = sqrt(s);
        L[j * 8 + j] = ljj;
        for (int i = j + 1; i < 8; ++i) {
            double t = S[i * 8 + j];
            for (int p = 0; p < j; ++p) t -= L[i * 8 + p] * L[j * 8 + p];
            L[i * 8 + j] = t / ljj;
        }
    }
}

/* ----------------------------------------------------------------- C10 --- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11): 10 rounds of
 *   (hi0, lo0) = M0 * c0, (hi1, lo1) = M1 * c2,
 *   c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0),
 * with the key bumped by the Weyl constants between rounds.                   */
void orc_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    }
    memcpy(out, c, sizeof(c));
}

/* uniform from the low 23 bits: u = (r mod 2^23 + 1/2) 2^-23 in [2^-24, 1 - 2^-24] (R13) */
static double u23(uint32_t r) { return ((double)(r & 0x7FFFFFu) + 0.5) * (1.0 / 8388608.0); }

static void bm_pair(uint32_t ra, uint32_t rb, double* z) {
    double ua = u23(ra), ub = u23(rb);
    double R = sqrt(-2.0 * log(ua));
    z[0] = R * cos(2.0 * ORC_PI * ub);
    z[1] = R * sin(2.0 * ORC_PI * ub);
}

/* key = (seed lo32, seed hi32); counters (cell lo32, iso_index, cell hi32, w) (R13; the paper
 * fixes no RNG).  Box-Muller pairs (u_a, u_b): R = sqrt(-2 ln u_a),
 * (R cos 2 pi u_b, R sin 2 pi u_b).
 * z0..z3 (R13c): sample s belongs to group g = 32 floor(s / 128) + (s mod 32) at position
 * t = floor(s / 32) mod 4; the group's word stream is the 12 words of the Philox blocks with
 * w = 2 (3 g + j), j = 0, 1, 2 (word i = word i mod 4 of block floor(i / 4)), and the sample
 * takes stream words 3t, 3t+1, 3t+2 = (A, B, C): (z0, z1) from (u(A), u(C)), (z2, z3) from
 * (u(B), u(D)), D = (A >> 24) | (B >> 24) << 8 | (C >> 24) << 16 -- four 23-bit uniforms from
 * disjoint bits of three words.
 * z4..z7: the block with w = 2s + 1, pairs (word 0, word 1) and (word 2, word 3).          */
void orc_normals8(uint64_t seed, int64_t cell, uint32_t iso_index, int64_t s, double* z) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const int64_t g = 32 * (s / 128) + s % 32, t = (s / 32) % 4;
    uint32_t w3[3];
    for (int i = 0; i < 3; ++i) {
        const int64_t wi = 3 * t + i;   /* stream word index */
        uint32_t ctr[4] = {(uint32_t)(uint64_t)cell, iso_index, (uint32_t)((uint64_t)cell >> 32),
                           (uint32_t)(2 * (3 * g + wi / 4))};
        uint32_t r[4];
        orc_philox4x32_10(ctr, key, r);
        w3[i] = r[wi % 4];
    }
    const uint32_t d = (w3[0] >> 24) | ((w3[1] >> 24) << 8) | ((w3[2] >> 24) << 16);
    bm_pair(w3[0], w3[2], z);
    bm_pair(w3[1], d, z + 2);
    uint32_t ctr[4] = {(uint32_t)(uint64_t)cell, iso_index, (uint32_t)((uint64_t)cell >> 32),
                       (uint32_t)(2 * s + 1)};
    uint32_t r[4];
    orc_philox4x32_10(ctr, key, r);
    bm_pair(r[0], r[1], z + 4);
    bm_pair(r[2], r[3], z + 6);
}

/* ----------------------------------------------------------------- C11 --- */
/* y = mu + L z; crossing = not(all y < theta) and not(all y > theta)
 * (the displayed sum at :130 is the NOT-crossed mass, R5). */
int64_t orc_mc_count(const double* mu, const double* L, double theta, int64_t n_samples,
                     uint64_t seed, int64_t cell, uint32_t iso_index) {
    int64_t count = 0;
    for (int64_t s = 0; s < n_samples; ++s) {
        double z[8], y[8];
        orc_normals8(seed, cell, iso_index, s, z);
        int below = 1, above = 1;
        for (int c = 0; c < 8; ++c) {
            y[c] = mu[c];
            for (int e = 0; e <= c; ++e) y[c] += L[c * 8 + e] * z[e];
            below = below && (y[c] < theta);
            above = above && (y[c] > theta);
        }
        if (!below && !above) ++count;
    }
    return count;
}

/* R13: the 8x8 factor is taken in the corner order PI8 = (0,3,5,6,1,2,4,7) --
 * the even-parity corners (a tetrahedron) first, then the odd ones -- and normal
 * z_i drives corner PI8[i]: y_PI8[i] = mu_PI8[i] + sum_{d<=i} L'_{id} z_d with
 * L' = chol(Sigma[PI8][PI8]).  Any square root of Sigma samples the same
 * 8-variate Gaussian; the crossing test is order-free. */
static const int PI8[8] = {0, 3, 5, 6, 1, 2, 4, 7};

int orc_pmc_cells(const orc_model_t* M, const int64_t* cells, int64_t n, double theta,
                  int64_t n_samples, uint64_t seed, uint32_t iso_index, double* lcp_out) {
    if (n_samples < 1) return ORC_EINVAL;
    int status = ORC_OK;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t q = 0; q < n; ++q) {
        double mu[8], cov[64], L[64], mup[8], covp[64];
        int st = orc_cell_posterior(M, cells[q], mu, cov);
        if (st != ORC_OK) {
#pragma omp critical
            status = st;
        }
        for (int i = 0; i < 8; ++i) {
            mup[i] = mu[PI8[i]];
            for (int j = 0; j < 8; ++j) covp[i * 8 + j] = cov[PI8[i] * 8 + PI8[j]];
        }
        orc_chol8(covp, L);
        lcp_out[q] = (double)orc_mc_count(mup, L, theta, n_samples, seed, cells[q], iso_index) /
                     (double)n_samples;
    }
    return status;
}

/* ---------------------------------------------------------------- NEXT-3 --- */
/* Fused multi-isovalue MC (the paper's isovalue sweep,
 * PAPER.md:346, :386): ONE sample stream per cell -- the counter word 1 is the
 * caller's `stream` index instead of a per-isovalue index (R27) -- and, for every
 * sample, the crossing test of C11 (ties cross, R24) applied
 * to each of the T isovalues.  counts_out[t] is therefore exactly
 * orc_mc_count(mu, L, thetas[t], N, seed, cell, stream). */
void orc_mc_count_multi(const double* mu, const double* L, const double* thetas, int32_t T,
                        int64_t n_samples, uint64_t seed, int64_t cell, uint32_t stream,
                        int64_t* counts_out) {
    for (int32_t t = 0; t < T; ++t) counts_out[t] = 0;
    for (int64_t s = 0; s < n_samples; ++s) {
        double z[8], y[8];
        orc_normals8(seed, cell, stream, s, z);
        for (int c = 0; c < 8; ++c) {
            y[c] = mu[c];
            for (int e = 0; e <= c; ++e) y[c] += L[c * 8 + e] * z[e];
        }
        for (int32_t t = 0; t < T; ++t) {
            int below = 1, above = 1;
            for (int c = 0; c < 8; ++c) {
                below = below && (y[c] < thetas[t]);
                above = above && (y[c] > thetas[t]);
            }
            if (!below && !above) ++counts_out[t];
        }
    }
}

/* Leaf pass for T isovalues on one cell list: posterior and chol8 once per cell
 * (they do not depend on theta), one sample stream, T counts.  mask[q] bit t
 * (NULL = all bits) says whether cell q is a leaf of isovalue t's octree; a
 * cleared bit gives LCP 0 (the cell was pruned for that isovalue).
 * lcp_out is T x n, isovalue-major. */
int orc_pmc_cells_multi(const orc_model_t* M, const int64_t* cells, int64_t n, const double* thetas,
                        int32_t T, const uint32_t* mask, int64_t n_samples, uint64_t seed,
                        uint32_t stream, double* lcp_out) {
    if (n_samples < 1 || T < 1 || T > 32) return ORC_EINVAL;
    int status = ORC_OK;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t q = 0; q < n; ++q) {
        double mu[8], cov[64], L[64], mup[8], covp[64];
        int64_t cnt[32];
        int st = orc_cell_posterior(M, cells[q], mu, cov);
        if (st != ORC_OK) {
#pragma omp critical
            status = st;
        }
        for (int i = 0; i < 8; ++i) {
            mup[i] = mu[PI8[i]];
            for (int j = 0; j < 8; ++j) covp[i * 8 + j] = cov[PI8[i] * 8 + PI8[j]];
        }
        orc_chol8(covp, L);
        orc_mc_count_multi(mup, L, thetas, T, n_samples, seed, cells[q], stream, cnt);
        for (int32_t t = 0; t < T; ++t) {
            int on = mask ? (int)((mask[q] >> t) & 1u) : 1;
            lcp_out[(int64_t)t * n + q] = on ? (double)cnt[t] / (double)n_samples : 0.0;
        }
    }
    return status;
}

/* ------------------------------------------------------------------ C6 --- */
/* P(Y < theta) = Phi((theta - mu) / sigma) (Sigma read as sigma, R4),
 * evaluated as erfc so that both tails keep full relative precision. */
void orc_tail_probs(double mu, double var, double theta, double* p_lo, double* p_hi) {
    double sd2 = sqrt(var) * ORC_SQRT2;
    *p_lo = 0.5 * erfc((mu - theta) / sd2);
    *p_hi = 0.5 * erfc((theta - mu) / sd2);
}

/* ---------------------------------------------------------------- NEXT-1 --- */
/* Gradient of the kernel w.r.t. its first argument a:
 * SE: dk/da_d = -k (a_d - b_d) / l_d^2;  Matern-5/2: -(5/3) s2 (1 + sqrt5 r) e^{-sqrt5 r} (a_d - b_d) / l_d^2. */
static void kernel_grad(const orc_kernel_t* kern, const double* a, const double* b, double* g) {
    double r2 = 0.0;
    for (int d = 0; d < 3; ++d) {
        double t = (a[d] - b[d]) / kern->lengthscale[d];
        r2 += t * t;
    }
    double c;
    if (kern->kind == 0) {
        c = -kern->variance * exp(-0.5 * r2);
    } else {
        double r = sqrt(r2), s5 = sqrt(5.0);
        c = -(5.0 / 3.0) * kern->variance * (1.0 + s5 * r) * exp(-s5 * r);
    }
    for (int d = 0; d < 3; ++d)
        g[d] = c * (a[d] - b[d]) / (kern->lengthscale[d] * kern->lengthscale[d]);
}

/* f(x) = (mu(x) - theta) / (sigma(x) sqrt 2) of bucket b's local GP and its gradient:
 * grad mu = sum_j grad k_j alpha_j; var = k(x,x) - v.v, v = L^-1 k_x;
 * grad var = -2 v . (L^-1 grad k); sigma = sqrt(max(var, floor)) (flat when floored). */
static double local_f_grad(const orc_model_t* M, int32_t b, const double* x, double theta, double* gf) {
    int ks = M->k, k = set_size(M, b);
    const int32_t* S = M->S + (size_t)b * ks;
    const double* L = M->L + (size_t)b * ks * ks;
    const double* al = M->alpha + (size_t)b * ks;
    double* kv = malloc(sizeof(double) * k * 4);
    double* v = malloc(sizeof(double) * k * 4);
    double mu = M->kern.prior_mean, gmu[3] = {0, 0, 0};
    for (int a = 0; a < k; ++a) {
        const double* xa = M->X + 3 * (size_t)S[a];
        double g[3];
        kv[a] = orc_kernel(&M->kern, x, xa);
        kernel_grad(&M->kern, x, xa, g);
        for (int d = 0; d < 3; ++d) kv[(d + 1) * k + a] = g[d];
        mu += kv[a] * al[a];
        for (int d = 0; d < 3; ++d) gmu[d] += g[d] * al[a];
    }
    for (int c = 0; c < 4; ++c) forward_sub(L, k, kv + (size_t)c * k, v + (size_t)c * k);
    double var = orc_kernel(&M->kern, x, x), gvar[3] = {0, 0, 0};
    for (int a = 0; a < k; ++a) {
        var -= v[a] * v[a];
        for (int d = 0; d < 3; ++d) gvar[d] -= 2.0 * v[a] * v[(d + 1) * k + a];
    }
    double fl = 1e-12 * M->kern.variance;
    double vf = var > fl ? var : fl, s = sqrt(vf);
    double f = (mu - theta) / (s * ORC_SQRT2);
    for (int d = 0; d < 3; ++d) {
        double gs = var > fl ? gvar[d] / (2.0 * s) : 0.0;
        gf[d] = (gmu[d] * s - (mu - theta) * gs) / (vf * ORC_SQRT2);
    }
    free(kv); free(v);
    return f;
}

/* R26: deterministic bounded search for the extreme of f over the node box,
 * maximising F = sgn * f from the lattice extreme `av` -- a projected limited-memory
 * quasi-Newton iteration in the spirit of the paper's L-BFGS-B (R26b):
 *   local model: the node's bucket when the node lies inside one bucket (level >=
 *   bucket_log2, the paper's per-node local model), else the start
 *   vertex's bucket with the box clipped to that bucket;
 *   direction: the free gradient g~ (components at an active bound that point out of
 *   the box are 0) times the L-BFGS inverse-Hessian estimate of -F (two-loop recursion
 *   over the last EXT_MEM pairs s = x+ - x, y = g - g+, kept when s.y > 1e-12 |s| |y|;
 *   H0 = (s.y / y.y) I), restricted to the free components; a non-ascent direction
 *   resets the memory and takes g~;
 *   step: x(t) = clip(x + t d), first t = step0 / |d| without memory (step0 = a quarter
 *   of the shortest box side), t = 1 with memory, t |d| <= the longest side;
 *   accept iff F(x(t)) > F and F(x(t)) >= F + 1e-4 g.(x(t) - x) (Armijo), else t /= 2;
 *   a step below 1e-12 of the longest side resets the memory, or ends the search
 *   without memory; so does a vanishing free gradient.
 * extreme_iters counts evaluations of f and grad f (one per trial point). */
#define EXT_MEM 4
static double extreme_search(const orc_model_t* M, double theta, int32_t level, const int64_t* base,
                             const int64_t* vmax, const int32_t* av, int sgn, double* f_start) {
    int64_t lo_v[3], hi_v[3];
    int32_t b;
    if (level >= M->b) {
        b = orc_vertex_bucket(M, (int32_t)base[0], (int32_t)base[1], (int32_t)base[2]);
        for (int d = 0; d < 3; ++d) { lo_v[d] = base[d]; hi_v[d] = vmax[d]; }
    } else {
        b = orc_vertex_bucket(M, av[0], av[1], av[2]);
        int32_t bi[3] = {b % M->nb[0], (b / M->nb[0]) % M->nb[1], b / (M->nb[0] * M->nb[1])};
        for (int d = 0; d < 3; ++d) {
            int64_t b0 = (int64_t)bi[d] * M->bs, b1 = b0 + M->bs;
            lo_v[d] = base[d] > b0 ? base[d] : b0;
            hi_v[d] = vmax[d] < b1 ? vmax[d] : b1;
        }
    }
    double blo[3], bhi[3], x[3], g[3];
    vertex_pos(M, (int32_t)lo_v[0], (int32_t)lo_v[1], (int32_t)lo_v[2], blo);
    vertex_pos(M, (int32_t)hi_v[0], (int32_t)hi_v[1], (int32_t)hi_v[2], bhi);
    vertex_pos(M, av[0], av[1], av[2], x);
    double mn = INFINITY, mx = 0.0;
    for (int d = 0; d < 3; ++d) {
        double w = bhi[d] - blo[d];
        if (w < mn) mn = w;
        if (w > mx) mx = w;
    }
    const double step0 = 0.25 * mn;
    double F = sgn * local_f_grad(M, b, x, theta, g);
    if (f_start) *f_start = sgn * F;
    for (int d = 0; d < 3; ++d) g[d] *= sgn;
    double S[EXT_MEM][3], Y[EXT_MEM][3], RHO[EXT_MEM];
    int nmem = 0;
    int need_dir = 1, done = 0;
    double dir[3] = {0, 0, 0}, t = 0.0, dn = 0.0;
    for (int it = 0; it < M->extreme_iters && !done; ++it) {
        double xt[3];
        for (;;) {                     /* find a trial point (no evaluation) */
            if (need_dir) {
                double gf[3];
                for (int d = 0; d < 3; ++d)
                    gf[d] = ((x[d] <= blo[d] && g[d] < 0.0) || (x[d] >= bhi[d] && g[d] > 0.0)) ? 0.0 : g[d];
                double gn = sqrt(gf[0] * gf[0] + gf[1] * gf[1] + gf[2] * gf[2]);
                if (!(gn > 0.0)) { done = 1; break; }
                /* two-loop recursion on the free gradient (newest pair last) */
                double q[3] = {gf[0], gf[1], gf[2]}, al[EXT_MEM];
                for (int i = nmem - 1; i >= 0; --i) {
                    al[i] = RHO[i] * (S[i][0] * q[0] + S[i][1] * q[1] + S[i][2] * q[2]);
                    for (int d = 0; d < 3; ++d) q[d] -= al[i] * Y[i][d];
                }
                if (nmem > 0) {
                    const int l = nmem - 1;
                    double sy = S[l][0] * Y[l][0] + S[l][1] * Y[l][1] + S[l][2] * Y[l][2];
                    double yy = Y[l][0] * Y[l][0] + Y[l][1] * Y[l][1] + Y[l][2] * Y[l][2];
                    for (int d = 0; d < 3; ++d) q[d] *= sy / yy;
                }
                for (int i = 0; i < nmem; ++i) {
                    double be = RHO[i] * (Y[i][0] * q[0] + Y[i][1] * q[1] + Y[i][2] * q[2]);
                    for (int d = 0; d < 3; ++d) q[d] += S[i][d] * (al[i] - be);
                }
                for (int d = 0; d < 3; ++d) dir[d] = gf[d] == 0.0 ? 0.0 : q[d];
                double slope = g[0] * dir[0] + g[1] * dir[1] + g[2] * dir[2];
                if (!(slope > 0.0)) {      /* not an ascent direction: reset to the gradient */
                    nmem = 0;
                    for (int d = 0; d < 3; ++d) dir[d] = gf[d];
                }
                dn = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
                t = nmem == 0 ? step0 / dn : 1.0;
                if (t * dn > mx) t = mx / dn;
                need_dir = 0;
            }
            if (t * dn < 1e-12 * mx) {     /* step collapsed */
                if (nmem > 0) { nmem = 0; need_dir = 1; continue; }
                done = 1;
                break;
            }
            for (int d = 0; d < 3; ++d) {
                double v = x[d] + t * dir[d];
                xt[d] = v < blo[d] ? blo[d] : (v > bhi[d] ? bhi[d] : v);
            }
            break;
        }
        if (done) break;
        double gt[3];
        double Ft = sgn * local_f_grad(M, b, xt, theta, gt);
        for (int d = 0; d < 3; ++d) gt[d] *= sgn;
        double gdx = g[0] * (xt[0] - x[0]) + g[1] * (xt[1] - x[1]) + g[2] * (xt[2] - x[2]);
        if (Ft > F && Ft >= F + 1e-4 * gdx) {
            double sv[3], yv[3];
            for (int d = 0; d < 3; ++d) { sv[d] = xt[d] - x[d]; yv[d] = g[d] - gt[d]; }
            double sy = sv[0] * yv[0] + sv[1] * yv[1] + sv[2] * yv[2];
            double ss = sqrt(sv[0] * sv[0] + sv[1] * sv[1] + sv[2] * sv[2]);
            double ys = sqrt(yv[0] * yv[0] + yv[1] * yv[1] + yv[2] * yv[2]);
            if (sy > 1e-12 * ss * ys) {
                if (nmem == EXT_MEM) {
                    for (int i = 1; i < EXT_MEM; ++i) {
                        for (int d = 0; d < 3; ++d) { S[i - 1][d] = S[i][d]; Y[i - 1][d] = Y[i][d]; }
                        RHO[i - 1] = RHO[i];
                    }
                    --nmem;
                }
                for (int d = 0; d < 3; ++d) { S[nmem][d] = sv[d]; Y[nmem][d] = yv[d]; }
                RHO[nmem] = 1.0 / sy;
                ++nmem;
            }
            F = Ft;
            for (int d = 0; d < 3; ++d) { x[d] = xt[d]; g[d] = gt[d]; }
            need_dir = 1;
        } else {
            t *= 0.5;
        }
    }
    return sgn * F;
}

void orc_model_set_extreme(orc_model_t* M, int32_t iters) { M->extreme_iters = iters > 0 ? iters : 0; }

/* test tap: out = {lattice zmax, lattice zmin, searched zmax, searched zmin, f at the two starts,
 * start of the max search (3), start of the min search (3)} */
void orc_node_extremes(const orc_model_t* M, double theta, int32_t level, int32_t i, int32_t j, int32_t k,
                       double* out) {
    int32_t h = M->lfull - level;
    int64_t side = (int64_t)1 << h, base[3], vmax[3];
    int32_t a[3] = {i, j, k};
    for (int d = 0; d < 3; ++d) {
        base[d] = (int64_t)a[d] * side;
        vmax[d] = base[d] + side < M->grid.cells[d] ? base[d] + side : M->grid.cells[d];
    }
    int32_t st = h - M->h_full > 0 ? h - M->h_full : 0;
    int64_t stride = (int64_t)1 << st;
    double zmax = -INFINITY, zmin = INFINITY;
    int32_t amax[3] = {0, 0, 0}, amin[3] = {0, 0, 0};
    for (int64_t vk = base[2];; vk = vk + stride < vmax[2] ? vk + stride : vmax[2]) {
        for (int64_t vj = base[1];; vj = vj + stride < vmax[1] ? vj + stride : vmax[1]) {
            for (int64_t vi = base[0];; vi = vi + stride < vmax[0] ? vi + stride : vmax[0]) {
                double xv[3], mu, var, vf = 0.0;
                vertex_pos(M, (int32_t)vi, (int32_t)vj, (int32_t)vk, xv);
                orc_local_marginal(M, orc_vertex_bucket(M, (int32_t)vi, (int32_t)vj, (int32_t)vk), xv, &mu, &var);
                floor_var(M, var, &vf);
                double zz = (mu - theta) / (sqrt(vf) * ORC_SQRT2);
                if (zz > zmax) { zmax = zz; amax[0] = (int32_t)vi; amax[1] = (int32_t)vj; amax[2] = (int32_t)vk; }
                if (zz < zmin) { zmin = zz; amin[0] = (int32_t)vi; amin[1] = (int32_t)vj; amin[2] = (int32_t)vk; }
                if (vi == vmax[0]) break;
            }
            if (vj == vmax[1]) break;
        }
        if (vk == vmax[2]) break;
    }
    out[0] = zmax;
    out[1] = zmin;
    out[2] = extreme_search(M, theta, level, base, vmax, amax, +1, &out[4]);
    out[3] = extreme_search(M, theta, level, base, vmax, amin, -1, &out[5]);
    vertex_pos(M, amax[0], amax[1], amax[2], out + 6);   /* the two search starts */
    vertex_pos(M, amin[0], amin[1], amin[2], out + 9);
}

double orc_local_f_grad(const orc_model_t* M, int32_t b, const double* x, double theta, double* grad) {
    return local_f_grad(M, b, x, theta, grad);
}

int orc_eval_node(const orc_model_t* M, double theta, double alpha, int32_t level,
                  int32_t i, int32_t j, int32_t k, orc_node_rec_t* rec) {
    int32_t h = M->lfull - level;
    int64_t side = (int64_t)1 << h;
    int32_t a[3] = {i, j, k};
    int64_t base[3], vmax[3];
    for (int d = 0; d < 3; ++d) {
        base[d] = (int64_t)a[d] * side;
        vmax[d] = base[d] + side < M->grid.cells[d] ? base[d] + side : M->grid.cells[d];
    }
    rec->level = level; rec->i = i; rec->j = j; rec->k = k;
    /* Alg. 1 lines 3-5: M~ = observations inside the node, p1 = max P(Y_i < theta),
     * p2 = max P(Y_i > theta) */
    int any = 0;
    double p1 = -1.0, p2 = -1.0;
    for (int32_t o = 0; o < M->m; ++o) {
        const int32_t* oc = M->obs_cell + 3 * o;
        int in = 1;
        for (int d = 0; d < 3; ++d) in = in && oc[d] >= base[d] && oc[d] < base[d] + side;
        if (!in) continue;
        double pl, ph;
        orc_tail_probs(M->mu_obs[o], M->var_obs[o], theta, &pl, &ph);
        if (!any || pl > p1) p1 = pl;
        if (!any || ph > p2) p2 = ph;
        any = 1;
    }
    rec->p1 = p1; rec->p2 = p2;
    if (any && p1 > alpha && p2 > alpha) {            /* case 1 (lines 6-7) */
        rec->ncase = 1; rec->U = 1.0; rec->refine = 1;
        return ORC_OK;
    }
    int ncase = !any ? 0 : (p2 <= alpha ? 2 : 3);     /* R8, R9 */
    /* B_l = min_D P(Y < theta), B_u = min_D P(Y > theta) over the candidate lattice
     * (R6): Q_lo = 1 - B_l, Q_hi = 1 - B_u. */
    int32_t st = h - M->h_full > 0 ? h - M->h_full : 0;
    int64_t stride = (int64_t)1 << st;
    int64_t lst[3][1 << 12];
    int nl[3];
    for (int d = 0; d < 3; ++d) {
        nl[d] = 0;
        for (int64_t v = base[d]; v < vmax[d]; v += stride) lst[d][nl[d]++] = v;
        lst[d][nl[d]++] = vmax[d];
    }
    /* z = (mu - theta) / (sigma sqrt 2): P(Y > theta) = erfc(-z)/2 and P(Y < theta) =
     * erfc(z)/2 are monotone in z, so Q_lo = max P(Y>theta) sits at max z and
     * Q_hi = max P(Y<theta) at min z (first occurrence wins ties). */
    double zmax = -INFINITY, zmin = INFINITY;
    int32_t amax[3] = {0, 0, 0}, amin[3] = {0, 0, 0};
    int status = ORC_OK;
    for (int z = 0; z < nl[2]; ++z)
        for (int y = 0; y < nl[1]; ++y)
            for (int x = 0; x < nl[0]; ++x) {
                int32_t vi = (int32_t)lst[0][x], vj = (int32_t)lst[1][y], vk = (int32_t)lst[2][z];
                double xv[3], mu, var, vf = 0.0;
                vertex_pos(M, vi, vj, vk, xv);
                orc_local_marginal(M, orc_vertex_bucket(M, vi, vj, vk), xv, &mu, &var);
                if (floor_var(M, var, &vf) != ORC_OK) status = ORC_ENUMERIC;
                double zz = (mu - theta) / (sqrt(vf) * ORC_SQRT2);
                if (zz > zmax) { zmax = zz; amax[0] = vi; amax[1] = vj; amax[2] = vk; }
                if (zz < zmin) { zmin = zz; amin[0] = vi; amin[1] = vj; amin[2] = vk; }
            }
    /* NEXT-1: refine the lattice extremes of coarse nodes by a
     * continuous bounded search of z over the node box (R26). */
    if (M->extreme_iters > 0 && h > M->h_full) {
        double zs = extreme_search(M, theta, level, base, vmax, amax, +1, NULL);
        if (zs > zmax) zmax = zs;
        zs = extreme_search(M, theta, level, base, vmax, amin, -1, NULL);
        if (zs < zmin) zmin = zs;
    }
    double q_lo = 0.5 * erfc(-zmax), q_hi = 0.5 * erfc(zmin);
    /* d = inclusive vertex count of the (clipped) node (Alg. 1 line 10, R7) */
    double dcount = (double)(vmax[0] - base[0] + 1) * (double)(vmax[1] - base[1] + 1) *
                    (double)(vmax[2] - base[2] + 1);
    double U;
    if (ncase == 2) {
        U = -expm1(dcount * log1p(-q_lo));                       /* 1 - B_l^d */
    } else if (ncase == 3) {
        U = -expm1(dcount * log1p(-q_hi));                       /* 1 - B_u^d */
    } else {
        U = -expm1(dcount * log1p(-q_lo)) - exp(dcount * log1p(-q_hi));   /* Eq. 4 */
        if (U < 0.0) U = 0.0;
        if (U > 1.0) U = 1.0;
    }
    rec->ncase = ncase; rec->U = U; rec->refine = U > alpha;
    return status;
}

/* ------------------------------------------------------------------ C7 --- */
typedef struct { int32_t i, j, k; } node3;

static int cmp64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

int orc_octree(const orc_model_t* M, double theta, double alpha, int32_t max_depth,
               int32_t sub_level, int32_t si, int32_t sj, int32_t sk,
               orc_node_rec_t** recs_out, int64_t* n_recs, int64_t** leaves_out, int64_t* n_leaves) {
    if (!(alpha > 0.0 && alpha < 0.5) || max_depth < 0 || max_depth > M->lfull) return ORC_EINVAL;
    int32_t L0 = sub_level >= 0 ? sub_level : 0;
    if (L0 > max_depth) return ORC_EINVAL;
    node3* front = malloc(sizeof(node3));
    int64_t nf = 1;
    front[0].i = sub_level >= 0 ? si : 0;
    front[0].j = sub_level >= 0 ? sj : 0;
    front[0].k = sub_level >= 0 ? sk : 0;
    int64_t cap_r = 1024, nr = 0, cap_l = 1024, nlv = 0;
    orc_node_rec_t* recs = malloc(sizeof(orc_node_rec_t) * cap_r);
    int64_t* leaves = malloc(sizeof(int64_t) * cap_l);
    int status = ORC_OK;
    const int32_t* cells = M->grid.cells;
    for (int32_t level = L0; level <= max_depth && nf > 0; ++level) {
        orc_node_rec_t* lr = malloc(sizeof(orc_node_rec_t) * nf);
#pragma omp parallel for schedule(dynamic)
        for (int64_t q = 0; q < nf; ++q) {
            int st = orc_eval_node(M, theta, alpha, level, front[q].i, front[q].j, front[q].k, &lr[q]);
            if (st != ORC_OK) {
#pragma omp critical
                status = st;
            }
        }
        if (nr + nf > cap_r) {
            while (nr + nf > cap_r) cap_r *= 2;
            recs = realloc(recs, sizeof(orc_node_rec_t) * cap_r);
        }
        memcpy(recs + nr, lr, sizeof(orc_node_rec_t) * nf);
        nr += nf;
        int32_t h = M->lfull - level;
        int64_t nn = 0;
        node3* next = malloc(sizeof(node3) * 8 * nf);
        for (int64_t q = 0; q < nf; ++q) {
            if (!lr[q].refine) continue;
            if (level < max_depth) {           /* Alg. 1 lines 14-21: 8 children */
                for (int c = 0; c < 8; ++c) {
                    node3 ch = {2 * front[q].i + (c & 1), 2 * front[q].j + ((c >> 1) & 1),
                                2 * front[q].k + (c >> 2)};
                    int64_t cs = (int64_t)1 << (h - 1);
                    if ((int64_t)ch.i * cs < cells[0] && (int64_t)ch.j * cs < cells[1] &&
                        (int64_t)ch.k * cs < cells[2])
                        next[nn++] = ch;
                }
            } else {                           /* lines 12-13: max depth, return the box's cells */
                int64_t side = (int64_t)1 << h;
                for (int64_t z = (int64_t)front[q].k * side; z < ((int64_t)front[q].k + 1) * side && z < cells[2]; ++z)
                    for (int64_t y = (int64_t)front[q].j * side; y < ((int64_t)front[q].j + 1) * side && y < cells[1]; ++y)
                        for (int64_t x = (int64_t)front[q].i * side; x < ((int64_t)front[q].i + 1) * side && x < cells[0]; ++x) {
                            if (nlv == cap_l) { cap_l *= 2; leaves = realloc(leaves, sizeof(int64_t) * cap_l); }
                            leaves[nlv++] = x + (int64_t)cells[0] * (y + (int64_t)cells[1] * z);
                        }
            }
        }
        free(lr);
        free(front);
        front = next;
        nf = nn;
    }
    free(front);
    qsort(leaves, nlv, sizeof(int64_t), cmp64);
    *recs_out = recs; *n_recs = nr; *leaves_out = leaves; *n_leaves = nlv;
    return status;
}

