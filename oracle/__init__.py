"""FP64 CPU oracle for the LCP hot path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  The product package
`paper_2512_12442_b200` never imports it, and the two share no code; the only
common module is `workloads` (seeded input generation, no method arithmetic).

The arithmetic lives in `lcp_oracle.c` (plain C, FP64, -ffp-contract=off);
this module is ctypes marshalling only.  Per-function citations are in the C
source.  Pins: tests/test_oracle_*.py (DESIGN.md §4 lists them).  Parity
unpinned parts: the coarse-level candidate-lattice extreme vs the
continuous regional extreme (R6), and the k-NN local-GP approximation error vs
the paper's beta-box local SGP (R2) -- neither has a value in PAPER.md.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lcp_oracle.c")
_LIB = os.path.join(_HERE, "liblcp_oracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle library in-tree (gcc, FP64, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "lcp_oracle.h"))):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Kernel(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("variance", C.c_double),
                ("lengthscale", C.c_double * 3), ("nugget", C.c_double),
                ("prior_mean", C.c_double)]


class Grid(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3), ("cells", C.c_int32 * 3),
                ("pad_", C.c_int32)]


NODE_DTYPE = np.dtype([("level", "<i4"), ("i", "<i4"), ("j", "<i4"), ("k", "<i4"),
                       ("ncase", "<i4"), ("refine", "<i4"), ("p1", "<f8"), ("p2", "<f8"),
                       ("U", "<f8")])

_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        dp = np.ctypeslib.ndpointer(np.float64, flags="C")
        ip64 = np.ctypeslib.ndpointer(np.int64, flags="C")
        ip32 = np.ctypeslib.ndpointer(np.int32, flags="C")
        up32 = np.ctypeslib.ndpointer(np.uint32, flags="C")
        P = C.c_void_p
        L.orc_kernel.restype = C.c_double
        L.orc_kernel.argtypes = [C.POINTER(Kernel), dp, dp]
        L.orc_gp_exact.argtypes = [C.POINTER(Kernel), dp, dp, C.c_int64, dp, C.c_int64, dp, P]
        L.orc_model_create.argtypes = [C.POINTER(Kernel), C.POINTER(Grid), dp, dp, C.c_int64,
                                       C.c_int32, C.c_int32, C.c_int32, C.POINTER(P)]
        L.orc_model_create_box.argtypes = [C.POINTER(Kernel), C.POINTER(Grid), dp, dp, C.c_int64,
                                           C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_int32, C.POINTER(P)]
        L.orc_model_destroy.argtypes = [P]
        L.orc_model_destroy.restype = None
        L.orc_model_nbuckets.argtypes = [P]
        L.orc_model_lfull.argtypes = [P]
        L.orc_model_bucket_set.argtypes = [P, C.c_int32, ip32]
        L.orc_model_bucket_set.restype = None
        L.orc_point_bucket.argtypes = [P, dp]
        L.orc_vertex_bucket.argtypes = [P, C.c_int32, C.c_int32, C.c_int32]
        L.orc_cell_bucket.argtypes = [P, C.c_int64]
        L.orc_local_marginal.argtypes = [P, C.c_int32, dp, C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]
        L.orc_cell_posterior.argtypes = [P, C.c_int64, dp, dp]
        L.orc_chol8.argtypes = [dp, dp]
        L.orc_chol8.restype = None
        L.orc_philox4x32_10.argtypes = [up32, up32, up32]
        L.orc_philox4x32_10.restype = None
        L.orc_normals8.argtypes = [C.c_uint64, C.c_int64, C.c_uint32, C.c_int64, dp]
        L.orc_normals8.restype = None
        L.orc_mc_count.restype = C.c_int64
        L.orc_mc_count.argtypes = [dp, dp, C.c_double, C.c_int64, C.c_uint64, C.c_int64,
                                   C.c_uint32]
        L.orc_pmc_cells.argtypes = [P, ip64, C.c_int64, C.c_double, C.c_int64, C.c_uint64,
                                    C.c_uint32, dp]
        L.orc_mc_count_multi.restype = None
        L.orc_mc_count_multi.argtypes = [dp, dp, dp, C.c_int32, C.c_int64, C.c_uint64, C.c_int64,
                                         C.c_uint32, ip64]
        L.orc_pmc_cells_multi.argtypes = [P, ip64, C.c_int64, dp, C.c_int32, P, C.c_int64,
                                          C.c_uint64, C.c_uint32, dp]
        L.orc_eval_node.argtypes = [P, C.c_double, C.c_double, C.c_int32, C.c_int32, C.c_int32,
                                    C.c_int32, P]
        L.orc_octree.argtypes = [P, C.c_double, C.c_double, C.c_int32, C.c_int32, C.c_int32,
                                 C.c_int32, C.c_int32, C.POINTER(P), C.POINTER(C.c_int64),
                                 C.POINTER(P), C.POINTER(C.c_int64)]
        L.orc_tail_probs.argtypes = [C.c_double, C.c_double, C.c_double,
                                     C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.orc_tail_probs.restype = None
        L.orc_model_set_extreme.argtypes = [P, C.c_int32]
        L.orc_model_set_extreme.restype = None
        L.orc_local_f_grad.restype = C.c_double
        L.orc_local_f_grad.argtypes = [P, C.c_int32, dp, C.c_double, dp]
        L.orc_node_extremes.argtypes = [P, C.c_double, C.c_int32, C.c_int32, C.c_int32, C.c_int32, dp]
        L.orc_node_extremes.restype = None
        L.orc_sgpr_exact.argtypes = [C.POINTER(Kernel), dp, dp, dp, C.c_int64, dp, C.c_int64, dp, P]
        L.orc_model_create_sgpr.argtypes = [C.POINTER(Kernel), C.POINTER(Grid), dp, dp, dp, C.c_int64,
                                            C.c_int32, C.c_int32, C.c_int32, C.POINTER(P)]
        L.orc_model_create_sgpr_mode.argtypes = [C.POINTER(Kernel), C.POINTER(Grid), dp, dp, dp, C.c_int64,
                                                 C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                                 C.POINTER(P)]
        L.orc_free.argtypes = [P]
        L.orc_free.restype = None
        L.orc_num_threads.restype = C.c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, status, what):
        super().__init__(f"oracle {what} failed with status {status}")
        self.status = status


def _check(st, what):
    if st != 0:
        raise OracleError(st, what)


def make_kernel(kind, variance, lengthscale, nugget, prior_mean=0.0) -> Kernel:
    ls = np.broadcast_to(np.asarray(lengthscale, dtype=np.float64), (3,))
    return Kernel(int(kind), 0, float(variance), (C.c_double * 3)(*ls), float(nugget),
                  float(prior_mean))


def make_grid(lo, hi, cells) -> Grid:
    return Grid((C.c_double * 3)(*lo), (C.c_double * 3)(*hi), (C.c_int32 * 3)(*cells), 0)


def kernel_value(kern: Kernel, a, b) -> float:
    return lib().orc_kernel(C.byref(kern), np.ascontiguousarray(a, np.float64),
                            np.ascontiguousarray(b, np.float64))


def gp_exact(kern: Kernel, X, y, Q, with_cov=True):
    X = np.ascontiguousarray(X, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    Q = np.ascontiguousarray(Q, np.float64).reshape(-1, 3)
    mu = np.zeros(len(Q))
    cov = np.zeros((len(Q), len(Q))) if with_cov else None
    _check(lib().orc_gp_exact(C.byref(kern), X, y, len(X), Q, len(Q),
                              mu, cov.ctypes.data if with_cov else None), "gp_exact")
    return mu, cov


def sgpr_exact(kern: Kernel, XM, muM, AM, Q, with_cov=True):
    """Eq. 1 of an SGPR model at query points Q."""
    XM = np.ascontiguousarray(XM, np.float64)
    muM = np.ascontiguousarray(muM, np.float64)
    AM = np.ascontiguousarray(AM, np.float64)
    Q = np.ascontiguousarray(Q, np.float64).reshape(-1, 3)
    mu = np.zeros(len(Q))
    cov = np.zeros((len(Q), len(Q))) if with_cov else None
    _check(lib().orc_sgpr_exact(C.byref(kern), XM, muM, AM, len(XM), Q, len(Q), mu,
                                cov.ctypes.data if with_cov else None), "sgpr_exact")
    return mu, cov


def philox4x32_10(ctr, key):
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(np.ascontiguousarray(ctr, np.uint32),
                            np.ascontiguousarray(key, np.uint32), out)
    return out


def normals8(seed, cell, iso_index, s):
    z = np.zeros(8)
    lib().orc_normals8(seed, cell, iso_index, s, z)
    return z


def chol8(S):
    L = np.zeros(64)
    lib().orc_chol8(np.ascontiguousarray(S, np.float64).reshape(64), L)
    return L.reshape(8, 8)


def mc_count(mu, L, theta, n_samples, seed, cell, iso_index=0):
    return lib().orc_mc_count(np.ascontiguousarray(mu, np.float64).reshape(8),
                              np.ascontiguousarray(L, np.float64).reshape(64), theta,
                              n_samples, seed, cell, iso_index)


def mc_count_multi(mu, L, thetas, n_samples, seed, cell, stream=0):
    th = np.ascontiguousarray(thetas, np.float64)
    out = np.zeros(len(th), np.int64)
    lib().orc_mc_count_multi(np.ascontiguousarray(mu, np.float64),
                             np.ascontiguousarray(np.asarray(L, np.float64).reshape(64)), th, len(th),
                             n_samples, seed, cell, stream, out)
    return out


def tail_probs(mu, var, theta):
    a, b = C.c_double(), C.c_double()
    lib().orc_tail_probs(mu, var, theta, C.byref(a), C.byref(b))
    return a.value, b.value


def num_threads() -> int:
    return lib().orc_num_threads()


class Model:
    """Bucket-local k-NN GP model (C3-C4) plus the oracle entry points that use it."""

    def __init__(self, kern: Kernel, grid: Grid, X, y, k, bucket_log2, h_full):
        self.kern, self.grid = kern, grid
        self.X = np.ascontiguousarray(X, np.float64)
        self.y = np.ascontiguousarray(y, np.float64)
        self.k = int(k)
        self.cells = tuple(grid.cells)
        h = C.c_void_p()
        _check(lib().orc_model_create(C.byref(kern), C.byref(grid), self.X, self.y, len(self.X),
                                      int(k), int(bucket_log2), int(h_full), C.byref(h)),
               "model_create")
        self._h = h

    @classmethod
    def sgpr(cls, kern: Kernel, grid: Grid, XM, muM, AM, k, bucket_log2, h_full, local_mode=0, beta=6.0):
        """NEXT-2: bucket-local SGPR model (Eq. 1 with the A_M term); local sets k-NN (0),
        beta-box (1) or capped beta-box (2)."""
        self = cls.__new__(cls)
        self.kern, self.grid = kern, grid
        self.X = np.ascontiguousarray(XM, np.float64)
        self.y = np.ascontiguousarray(muM, np.float64)
        self.A = np.ascontiguousarray(AM, np.float64)
        self.k = int(k)
        self.cells = tuple(grid.cells)
        h = C.c_void_p()
        _check(lib().orc_model_create_sgpr_mode(C.byref(kern), C.byref(grid), self.X, self.y, self.A, len(self.X),
                                                int(k), int(bucket_log2), int(h_full), int(local_mode), float(beta),
                                                C.byref(h)), "model_create_sgpr")
        self._h = h
        return self

    @classmethod
    def box(cls, kern: Kernel, grid: Grid, X, y, k, bucket_log2, h_full, beta, cap=False):
        """R28 (NEXT-2): local set = observations in the bucket box enlarged by beta l_d;
        cap (R28b): a box holding more than k observations gives the bucket its k-NN set."""
        self = cls.__new__(cls)
        self.kern, self.grid = kern, grid
        self.X = np.ascontiguousarray(X, np.float64)
        self.y = np.ascontiguousarray(y, np.float64)
        self.k = int(k)
        self.cells = tuple(grid.cells)
        h = C.c_void_p()
        _check(lib().orc_model_create_box(C.byref(kern), C.byref(grid), self.X, self.y, len(self.X), int(k),
                                          int(bucket_log2), int(h_full), float(beta), int(bool(cap)), C.byref(h)),
               "model_create_box")
        self._h = h
        return self

    @classmethod
    def from_config(cls, cfg, X, y, k=None, bucket_log2=None, h_full=None):
        kern = make_kernel(cfg.kernel, cfg.variance, cfg.lengthscale, cfg.nugget, cfg.prior_mean)
        grid = make_grid(cfg.lo, cfg.hi, cfg.cells)
        return cls(kern, grid, X, y, cfg.k if k is None else k,
                   cfg.bucket_log2 if bucket_log2 is None else bucket_log2,
                   cfg.h_full if h_full is None else h_full)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_model_destroy(self._h)
            self._h = None

    @property
    def nbuckets(self):
        return lib().orc_model_nbuckets(self._h)

    @property
    def lfull(self):
        return lib().orc_model_lfull(self._h)

    def bucket_set(self, b):
        out = np.zeros(self.k, np.int32)
        lib().orc_model_bucket_set(self._h, b, out)
        return out

    def point_bucket(self, x):
        return lib().orc_point_bucket(self._h, np.ascontiguousarray(x, np.float64))

    def vertex_bucket(self, i, j, k):
        return lib().orc_vertex_bucket(self._h, i, j, k)

    def cell_bucket(self, cell):
        return lib().orc_cell_bucket(self._h, int(cell))

    def local_marginal(self, b, x):
        mu, var = C.c_double(), C.c_double()
        _check(lib().orc_local_marginal(self._h, b, np.ascontiguousarray(x, np.float64),
                                        C.byref(mu), C.byref(var)), "local_marginal")
        return mu.value, var.value

    def set_extreme(self, iters):
        """NEXT-1 (R26): continuous extreme search iterations at nodes with h > h_full."""
        lib().orc_model_set_extreme(self._h, int(iters))

    def f_grad(self, b, x, theta):
        g = np.zeros(3)
        f = lib().orc_local_f_grad(self._h, b, np.ascontiguousarray(x, np.float64), theta, g)
        return f, g

    def node_extremes(self, theta, level, i, j, k, starts=False):
        out = np.zeros(12)
        lib().orc_node_extremes(self._h, theta, level, i, j, k, out)
        return (out[:6], out[6:9], out[9:12]) if starts else out[:6]

    def cell_posterior(self, cell):
        mu = np.zeros(8)
        cov = np.zeros(64)
        _check(lib().orc_cell_posterior(self._h, int(cell), mu, cov), "cell_posterior")
        return mu, cov.reshape(8, 8)

    def pmc_cells(self, cells, theta, n_samples, seed, iso_index=0):
        cells = np.ascontiguousarray(cells, np.int64)
        out = np.zeros(len(cells))
        _check(lib().orc_pmc_cells(self._h, cells, len(cells), theta, n_samples, seed,
                                   iso_index, out), "pmc_cells")
        return out

    def pmc_cells_multi(self, cells, thetas, n_samples, seed, stream=0, mask=None):
        """NEXT-3 (R27): T x n LCP, one sample stream for all isovalues; mask[q] bit t
        marks cell q as a leaf of isovalue t (None = all)."""
        cells = np.ascontiguousarray(cells, np.int64)
        th = np.ascontiguousarray(thetas, np.float64)
        out = np.zeros(len(th) * len(cells))
        mk = None if mask is None else np.ascontiguousarray(mask, np.uint32)
        _check(lib().orc_pmc_cells_multi(self._h, cells, len(cells), th, len(th),
                                         None if mk is None else mk.ctypes.data, n_samples, seed,
                                         stream, out), "pmc_cells_multi")
        return out.reshape(len(th), len(cells))

    def eval_node(self, theta, alpha, level, i, j, k):
        rec = np.zeros(1, NODE_DTYPE)
        _check(lib().orc_eval_node(self._h, theta, alpha, level, i, j, k, rec.ctypes.data),
               "eval_node")
        return rec[0]

    def octree(self, theta, alpha, max_depth, subtree=None):
        """Returns (records structured array, sorted leaf cell ids)."""
        rp, nr, lp, nl = C.c_void_p(), C.c_int64(), C.c_void_p(), C.c_int64()
        sl, si, sj, sk = subtree if subtree is not None else (-1, 0, 0, 0)
        _check(lib().orc_octree(self._h, theta, alpha, max_depth, sl, si, sj, sk, C.byref(rp),
                                C.byref(nr), C.byref(lp), C.byref(nl)), "octree")
        try:
            recs = np.frombuffer((C.c_char * (nr.value * NODE_DTYPE.itemsize)).from_address(
                rp.value), dtype=NODE_DTYPE).copy() if nr.value else np.zeros(0, NODE_DTYPE)
            leaves = np.frombuffer((C.c_char * (nl.value * 8)).from_address(lp.value),
                                   dtype=np.int64).copy() if nl.value else np.zeros(0, np.int64)
        finally:
            lib().orc_free(rp)
            lib().orc_free(lp)
        return recs, leaves
