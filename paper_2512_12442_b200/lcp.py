"""Thin ctypes binding of liblcp.so (include/lcp.h) -- argument marshalling only.

Every step of the path runs in the library's sm_100a kernels; this module only
moves pointers and sizes across the C ABI.  torch is used for device memory,
streams and process groups.  There is no CPU fallback: importing works without
a GPU, but `Context(...)` raises when liblcp.so or a CUDA device is missing.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LCP_LIB", os.path.join(_HERE, "liblcp.so"))

LCP_OK, LCP_EINVAL, LCP_ESTATE, LCP_EFACTOR, LCP_ENUMERIC, LCP_ECUDA, LCP_ENOMEM = range(7)
STATUS_NAMES = {0: "LCP_OK", 1: "LCP_EINVAL", 2: "LCP_ESTATE", 3: "LCP_EFACTOR", 4: "LCP_ENUMERIC",
                5: "LCP_ECUDA", 6: "LCP_ENOMEM"}
K_SE, K_MATERN52 = 0, 1
FP64, FP32 = 0, 1

# every symbol include/lcp.h declares
EXPORTS = ["lcp_create", "lcp_destroy", "lcp_last_error", "lcp_fit_local", "lcp_octree_refine",
           "lcp_pmc_cells", "lcp_scatter_field", "lcp_run_field", "lcp_node_records",
           "lcp_cell_posterior", "lcp_point_marginals", "lcp_bucket_sets", "lcp_get_info",
           "lcp_stats_json", "lcp_synchronize", "lcp_set_level_field", "lcp_fit_sgpr",
           "lcp_pmc_cells_multi", "lcp_run_field_multi", "lcp_union_cells", "lcp_slab_auto_level",
           "lcp_slab_cuts", "lcp_fit_shard_buffers", "lcp_fit_finish"]


class LcpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class KernelT(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("variance", C.c_double),
                ("lengthscale", C.c_double * 3), ("nugget", C.c_double), ("prior_mean", C.c_double)]


class GridT(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3), ("cells", C.c_int32 * 3),
                ("pad_", C.c_int32)]


class OptsT(C.Structure):
    _fields_ = [("bucket_log2", C.c_int32), ("h_full", C.c_int32), ("precision", C.c_int32),
                ("slab_rank", C.c_int32), ("slab_count", C.c_int32), ("slab_level", C.c_int32),
                ("keep_records", C.c_int32), ("extreme_iters", C.c_int32), ("brick_pass", C.c_int32),
                ("local_mode", C.c_int32), ("fit_shard", C.c_int32), ("beta", C.c_double)]


class InfoT(C.Structure):
    _fields_ = [("m", C.c_int64), ("k", C.c_int32), ("nbuckets", C.c_int32), ("nb", C.c_int32 * 3),
                ("lfull", C.c_int32), ("bucket_side", C.c_int32), ("device", C.c_int32)]


NODE_DTYPE = np.dtype([("level", "<i4"), ("i", "<i4"), ("j", "<i4"), ("k", "<i4"),
                       ("ncase", "<i4"), ("refine", "<i4"), ("p1", "<f8"), ("p2", "<f8"),
                       ("U", "<f8")])

_lib = None


def load_library() -> C.CDLL:
    """Load liblcp.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"liblcp.so not built at {LIB_PATH}; run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P, i32, i64, u32, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
    L.lcp_create.argtypes = [i32, P, C.POINTER(P)]
    L.lcp_destroy.argtypes = [P]
    L.lcp_destroy.restype = None
    L.lcp_last_error.argtypes = [P]
    L.lcp_last_error.restype = C.c_char_p
    L.lcp_fit_local.argtypes = [P, P, P, i64, i32, C.POINTER(KernelT), i32, C.POINTER(GridT),
                                C.POINTER(OptsT)]
    L.lcp_octree_refine.argtypes = [P, dbl, dbl, i32, C.POINTER(i64), C.POINTER(P)]
    L.lcp_pmc_cells.argtypes = [P, P, i64, i32, dbl, i64, u64, u32, P, i32]
    L.lcp_scatter_field.argtypes = [P, P, P, i64, P]
    L.lcp_run_field.argtypes = [P, dbl, dbl, i32, i64, u64, u32, P, i32, C.POINTER(i64)]
    L.lcp_node_records.argtypes = [P, C.POINTER(i64), C.POINTER(P)]
    L.lcp_cell_posterior.argtypes = [P, P, i64, P, P]
    L.lcp_point_marginals.argtypes = [P, P, i64, P, P, P]
    L.lcp_bucket_sets.argtypes = [P, P]
    L.lcp_get_info.argtypes = [P, C.POINTER(InfoT)]
    L.lcp_stats_json.argtypes = [P, C.c_char_p, C.c_size_t]
    L.lcp_synchronize.argtypes = [P]
    L.lcp_set_level_field.argtypes = [P, P]
    L.lcp_fit_sgpr.argtypes = [P, P, P, P, i64, i32, C.POINTER(KernelT), i32, C.POINTER(GridT),
                               C.POINTER(OptsT)]
    L.lcp_pmc_cells_multi.argtypes = [P, P, i64, P, i32, P, i64, u64, u32, P]
    L.lcp_run_field_multi.argtypes = [P, P, i32, dbl, i32, i64, u64, u32, P, i32, P, C.POINTER(i64)]
    L.lcp_union_cells.argtypes = [P, C.POINTER(i64), C.POINTER(P), C.POINTER(P)]
    L.lcp_slab_auto_level.argtypes = [C.POINTER(GridT), i32, i32]
    L.lcp_fit_shard_buffers.argtypes = [P, C.POINTER(P), C.POINTER(i64), C.POINTER(P), C.POINTER(i64)]
    L.lcp_fit_finish.argtypes = [P]
    L.lcp_slab_cuts.argtypes = [P, i32, i32, P]
    for name in EXPORTS:
        if name not in ("lcp_destroy", "lcp_last_error"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _is_dev(t) -> int:
    return 0 if isinstance(t, np.ndarray) else int(t.is_cuda)


class Context:
    """One lcp_ctx_t on one CUDA device (see include/lcp.h for every call)."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        self._L = load_library()
        self.device = device
        self._torch = torch
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        h = C.c_void_p()
        st = self._L.lcp_create(device, C.c_void_p(stream.cuda_stream), C.byref(h))
        if st != LCP_OK:
            raise LcpError(st, f"lcp_create(device={device}) failed (no CUDA device?)")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._L.lcp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what):
        if st != LCP_OK:
            raise LcpError(st, f"{what}: {self._L.lcp_last_error(self._h).decode()}")

    # -- a1-a4
    def fit_local(self, xyz, y, kernel: Tuple, k: int, grid: Tuple, bucket_log2: int = 0,
                  h_full: int = 2, precision: int = FP64, slab_rank: int = 0, slab_count: int = 1,
                  slab_level: int = 0, keep_records=False, extreme_iters: int = 0, brick_pass: int = 0,
                  local_mode: int = 0, beta: float = 6.0, fit_shard: int = 0):
        """xyz (m,3) / y (m,) float64, either torch CUDA tensors or numpy host arrays.
        kernel = (kind, variance, lengthscale[3], nugget, prior_mean); grid = (lo, hi, cells).
        keep_records: True = every level, int L = levels < L (parity tap)."""
        if keep_records is True:
            keep_records = 64
        kind, var, ls, nug, m0 = kernel
        ls = list(np.broadcast_to(np.asarray(ls, dtype=np.float64), (3,)))
        kt = KernelT(int(kind), 0, float(var), (C.c_double * 3)(*ls), float(nug), float(m0))
        lo, hi, cells = grid
        gt = GridT((C.c_double * 3)(*lo), (C.c_double * 3)(*hi), (C.c_int32 * 3)(*cells), 0)
        ot = OptsT(bucket_log2, h_full, precision, slab_rank, slab_count, slab_level,
                   int(keep_records), int(extreme_iters), int(brick_pass), int(local_mode), int(fit_shard),
                   float(beta))
        if isinstance(xyz, np.ndarray):
            xyz = np.ascontiguousarray(xyz, np.float64)
            y = np.ascontiguousarray(y, np.float64)
        else:
            assert xyz.dtype == self._torch.float64 and xyz.is_contiguous() and y.is_contiguous()
        self._keep = (xyz, y)
        st = self._L.lcp_fit_local(self._h, C.c_void_p(_ptr(xyz)), C.c_void_p(_ptr(y)), len(y),
                                   _is_dev(xyz), C.byref(kt), int(k), C.byref(gt), C.byref(ot))
        self._check(st, "lcp_fit_local")
        self.grid = (tuple(lo), tuple(hi), tuple(cells))
        self._slab_count = slab_count
        return self

    def fit_shard_buffers(self):
        """Sharded fit: (bdata, sets) as uint8 CUDA tensor views of the ctx-owned arrays (no
        copy) and their per-rank chunk sizes in bytes, for an in-place all-gather."""
        pb, ps = C.c_void_p(), C.c_void_p()
        nb, ns = C.c_int64(), C.c_int64()
        self._check(self._L.lcp_fit_shard_buffers(self._h, C.byref(pb), C.byref(nb), C.byref(ps), C.byref(ns)),
                    "lcp_fit_shard_buffers")
        return self._view_dev(pb.value, nb.value), nb.value, self._view_dev(ps.value, ns.value), ns.value

    def _view_dev(self, ptr, chunk):
        """uint8 CUDA tensor aliasing slab_count x chunk bytes of a ctx-owned device array."""
        torch = self._torch
        n = chunk * self._slab_count

        class _View:
            __cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                        "strides": None, "stream": None}

        with torch.cuda.device(self.device):
            return torch.as_tensor(_View(), device=f"cuda:{self.device}")

    def fit_finish(self):
        self._check(self._L.lcp_fit_finish(self._h), "lcp_fit_finish")
        return self

    def fit_sgpr(self, xyz_M, mu_M, A_M, kernel: Tuple, k: int, grid: Tuple, bucket_log2: int = 0,
                 h_full: int = 2, keep_records=False, extreme_iters: int = 0, local_mode: int = 0,
                 beta: float = 6.0):
        """NEXT-2: bucket-local Eq. 1 of an SGPR model (inducing points, mean, covariance A_M);
        local sets k-NN (local_mode 0), beta-box (1) or beta-box capped at k (2)."""
        if keep_records is True:
            keep_records = 64
        kind, var, ls, nug, m0 = kernel
        ls = list(np.broadcast_to(np.asarray(ls, dtype=np.float64), (3,)))
        kt = KernelT(int(kind), 0, float(var), (C.c_double * 3)(*ls), float(nug), float(m0))
        lo, hi, cells = grid
        gt = GridT((C.c_double * 3)(*lo), (C.c_double * 3)(*hi), (C.c_int32 * 3)(*cells), 0)
        ot = OptsT(bucket_log2, h_full, FP64, 0, 1, 0, int(keep_records), int(extreme_iters), 0, int(local_mode), 0,
                   float(beta))
        if isinstance(xyz_M, np.ndarray):
            xyz_M = np.ascontiguousarray(xyz_M, np.float64)
            mu_M = np.ascontiguousarray(mu_M, np.float64)
            A_M = np.ascontiguousarray(A_M, np.float64)
        self._keep = (xyz_M, mu_M, A_M)
        st = self._L.lcp_fit_sgpr(self._h, C.c_void_p(_ptr(xyz_M)), C.c_void_p(_ptr(mu_M)),
                                  C.c_void_p(_ptr(A_M)), len(mu_M), _is_dev(xyz_M), C.byref(kt), int(k),
                                  C.byref(gt), C.byref(ot))
        self._check(st, "lcp_fit_sgpr")
        self.grid = (tuple(lo), tuple(hi), tuple(cells))
        return self

    # -- a5-a6
    def octree_refine(self, isovalue: float, threshold: float, max_depth: int):
        """Returns a torch int64 CUDA tensor VIEW of the ctx-owned leaf list (copy it to keep)."""
        n = C.c_int64()
        p = C.c_void_p()
        st = self._L.lcp_octree_refine(self._h, float(isovalue), float(threshold), int(max_depth),
                                       C.byref(n), C.byref(p))
        self._check(st, "lcp_octree_refine")
        return self._wrap_dev(p.value, n.value, self._torch.int64)

    def _wrap_dev(self, ptr, n, dtype):
        """Copy n elements of a ctx-owned device array into a fresh torch tensor."""
        torch = self._torch
        if n == 0 or not ptr:
            return torch.empty(0, dtype=dtype, device=f"cuda:{self.device}")
        typestr = {torch.int64: "<i8", torch.uint8: "|u1", torch.float32: "<f4",
                   torch.float64: "<f8"}[dtype]

        class _View:
            __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                        "version": 3, "strides": None, "stream": None}

        with torch.cuda.device(self.device):
            return torch.as_tensor(_View(), device=f"cuda:{self.device}").clone()

    # -- a7-a8
    def pmc_cells(self, cells, isovalue: float, n_samples: int, seed: int, iso_index: int = 0,
                  out=None):
        torch = self._torch
        n = len(cells)
        if out is None:
            out = torch.empty(n, dtype=torch.float32, device=cells.device if not isinstance(
                cells, np.ndarray) else f"cuda:{self.device}")
        st = self._L.lcp_pmc_cells(self._h, C.c_void_p(_ptr(cells)), n, _is_dev(cells),
                                   float(isovalue), int(n_samples), int(seed), int(iso_index),
                                   C.c_void_p(_ptr(out)), _is_dev(out))
        self._check(st, "lcp_pmc_cells")
        return out

    # -- a9
    def scatter_field(self, cells, lcp, field=None):
        torch = self._torch
        if field is None:
            nx, ny, nz = self.grid[2]
            field = torch.empty(nx * ny * nz, dtype=torch.float32, device=f"cuda:{self.device}")
        st = self._L.lcp_scatter_field(self._h, C.c_void_p(_ptr(cells)), C.c_void_p(_ptr(lcp)),
                                       len(cells), C.c_void_p(_ptr(field)))
        self._check(st, "lcp_scatter_field")
        return field

    def run_field(self, isovalue, threshold, max_depth, n_samples, seed, iso_index=0, field=None):
        torch = self._torch
        if field is None:
            nx, ny, nz = self.grid[2]
            field = torch.empty(nx * ny * nz, dtype=torch.float32, device=f"cuda:{self.device}")
        n = C.c_int64()
        st = self._L.lcp_run_field(self._h, float(isovalue), float(threshold), int(max_depth),
                                   int(n_samples), int(seed), int(iso_index), C.c_void_p(_ptr(field)),
                                   _is_dev(field), C.byref(n))
        self._check(st, "lcp_run_field")
        return field, n.value

    # -- NEXT-3: fused multi-isovalue leaf pass
    def pmc_cells_multi(self, cells, isovalues: Sequence[float], n_samples: int, seed: int, stream: int = 0,
                        mask=None, out=None):
        """(T, n) float32 CUDA tensor: one sample stream per cell, every isovalue tested.
        cells: int64 CUDA tensor; mask: uint32-valued CUDA tensor (int32 storage) or None."""
        torch = self._torch
        th = np.ascontiguousarray(isovalues, np.float64)
        n = len(cells)
        if out is None:
            out = torch.empty((len(th), n), dtype=torch.float32, device=cells.device)
        st = self._L.lcp_pmc_cells_multi(self._h, C.c_void_p(_ptr(cells)), n, C.c_void_p(th.ctypes.data),
                                         len(th), C.c_void_p(_ptr(mask)), int(n_samples), int(seed),
                                         int(stream), C.c_void_p(_ptr(out)))
        self._check(st, "lcp_pmc_cells_multi")
        return out

    def run_field_multi(self, isovalues: Sequence[float], threshold, max_depth, n_samples, seed, stream=0,
                        fields=None):
        """Returns (fields (T, nx*ny*nz) float32, leaf counts per isovalue, union size)."""
        torch = self._torch
        th = np.ascontiguousarray(isovalues, np.float64)
        if fields is None:
            nx, ny, nz = self.grid[2]
            fields = torch.empty((len(th), nx * ny * nz), dtype=torch.float32, device=f"cuda:{self.device}")
        nl = np.zeros(len(th), np.int64)
        nu = C.c_int64()
        st = self._L.lcp_run_field_multi(self._h, C.c_void_p(th.ctypes.data), len(th), float(threshold),
                                         int(max_depth), int(n_samples), int(seed), int(stream),
                                         C.c_void_p(_ptr(fields)), _is_dev(fields), C.c_void_p(nl.ctypes.data),
                                         C.byref(nu))
        self._check(st, "lcp_run_field_multi")
        return fields, nl, nu.value

    def union_cells(self):
        """(cells int64, mask int64) of the last run_field_multi (copies)."""
        n = C.c_int64()
        pc, pm = C.c_void_p(), C.c_void_p()
        self._check(self._L.lcp_union_cells(self._h, C.byref(n), C.byref(pc), C.byref(pm)), "lcp_union_cells")
        cells = self._wrap_dev(pc.value, n.value, self._torch.int64)
        raw = self._wrap_dev(pm.value, 4 * n.value, self._torch.uint8)
        mask = raw.view(self._torch.int32).to(self._torch.int64) & 0xFFFFFFFF if n.value else raw.to(
            self._torch.int64)
        return cells, mask

    def set_level_field(self, level=None):
        """NEXT-4: register a torch uint8 CUDA tensor (nx*ny*nz) that every later
        refine fills with the octree level at which each cell stopped."""
        self._level = level
        self._check(self._L.lcp_set_level_field(self._h, C.c_void_p(_ptr(level))), "lcp_set_level_field")
        return level

    # -- parity taps
    def node_records(self) -> np.ndarray:
        n = C.c_int64()
        p = C.c_void_p()
        self._check(self._L.lcp_node_records(self._h, C.byref(n), C.byref(p)), "lcp_node_records")
        raw = self._wrap_dev(p.value, n.value * NODE_DTYPE.itemsize, self._torch.uint8)
        return raw.cpu().numpy().view(NODE_DTYPE)

    def node_records_device(self):
        """The node records of the last refine as a raw uint8 CUDA tensor (a copy;
        view it as int32 (n, 12): level, i, j, k, case, refine, then p1, p2, U as FP64)."""
        n = C.c_int64()
        p = C.c_void_p()
        self._check(self._L.lcp_node_records(self._h, C.byref(n), C.byref(p)), "lcp_node_records")
        return self._wrap_dev(p.value, n.value * NODE_DTYPE.itemsize, self._torch.uint8)

    def cell_posterior(self, cells):
        torch = self._torch
        n = len(cells)
        mu = torch.empty((n, 8), dtype=torch.float64, device=cells.device)
        cov = torch.empty((n, 8, 8), dtype=torch.float64, device=cells.device)
        self._check(self._L.lcp_cell_posterior(self._h, C.c_void_p(_ptr(cells)), n,
                                               C.c_void_p(_ptr(mu)), C.c_void_p(_ptr(cov))),
                    "lcp_cell_posterior")
        return mu, cov

    def point_marginals(self, xyz, buckets=None):
        torch = self._torch
        n = xyz.shape[0]
        mu = torch.empty(n, dtype=torch.float64, device=xyz.device)
        var = torch.empty(n, dtype=torch.float64, device=xyz.device)
        self._check(self._L.lcp_point_marginals(self._h, C.c_void_p(_ptr(xyz)), n,
                                                C.c_void_p(_ptr(buckets)), C.c_void_p(_ptr(mu)),
                                                C.c_void_p(_ptr(var))), "lcp_point_marginals")
        return mu, var

    def info(self) -> dict:
        i = InfoT()
        self._check(self._L.lcp_get_info(self._h, C.byref(i)), "lcp_get_info")
        return {"m": i.m, "k": i.k, "nbuckets": i.nbuckets, "nb": tuple(i.nb), "lfull": i.lfull,
                "bucket_side": i.bucket_side, "device": i.device}

    def bucket_sets(self):
        torch = self._torch
        inf = self.info()
        out = torch.empty((inf["nbuckets"], inf["k"]), dtype=torch.int32, device=f"cuda:{self.device}")
        self._check(self._L.lcp_bucket_sets(self._h, C.c_void_p(_ptr(out))), "lcp_bucket_sets")
        return out

    def stats(self) -> dict:
        buf = C.create_string_buffer(1 << 16)
        self._check(self._L.lcp_stats_json(self._h, buf, len(buf)), "lcp_stats_json")
        return json.loads(buf.value.decode())

    def synchronize(self):
        self._check(self._L.lcp_synchronize(self._h), "lcp_synchronize")


def slab_auto_level(cells, slab_count: int, max_depth: int) -> int:
    """lcp_slab_auto_level (host-only): the slab level refine picks for slab_count ranks."""
    gt = GridT((C.c_double * 3)(0, 0, 0), (C.c_double * 3)(1, 1, 1), (C.c_int32 * 3)(*cells), 0)
    lv = load_library().lcp_slab_auto_level(C.byref(gt), int(slab_count), int(max_depth))
    if lv < 0:
        raise LcpError(LCP_EINVAL, "lcp_slab_auto_level: bad arguments")
    return lv


def slab_cuts(weights, slab_count: int) -> np.ndarray:
    """lcp_slab_cuts (host-only): layer cuts (slab_count + 1) balancing the weights."""
    w = np.ascontiguousarray(weights, np.int64)
    out = np.zeros(slab_count + 1, np.int32)
    st = load_library().lcp_slab_cuts(C.c_void_p(w.ctypes.data), len(w), int(slab_count), C.c_void_p(out.ctypes.data))
    if st != LCP_OK:
        raise LcpError(st, "lcp_slab_cuts: bad arguments")
    return out


def config_args(cfg, k=None, bucket_log2=None):
    """(kernel, grid, k, bucket_log2, h_full) tuples for a workloads.Config."""
    kernel = (cfg.kernel, cfg.variance, cfg.lengthscale, cfg.nugget, cfg.prior_mean)
    grid = (cfg.lo, cfg.hi, cfg.cells)
    return kernel, grid, (cfg.k if k is None else k), (cfg.bucket_log2 if bucket_log2 is None
                                                        else bucket_log2), cfg.h_full
