"""Comparison helpers for GPU-vs-oracle parity (DESIGN.md §2 R18, R19)."""
from __future__ import annotations

import numpy as np

BAND = 1e-6


def posterior_close(mu_g, mu_o, cov_g, cov_o, sigma2, tau):
    """R18: |dmu| <= tau max(|mu|, sigma_f), |dSigma| <= tau max(|Sigma|, sigma_f^2)."""
    sf = np.sqrt(sigma2)
    emu = np.abs(mu_g - mu_o) / np.maximum(np.abs(mu_o), sf)
    ecov = np.abs(cov_g - cov_o) / np.maximum(np.abs(cov_o), sigma2)
    return float(emu.max(initial=0.0)), float(ecov.max(initial=0.0))


def node_keys(rec):
    """(level, i, j, k) packed into one int64: level << 60 | k << 40 | j << 20 | i."""
    return ((rec["level"].astype(np.int64) << 60) | (rec["k"].astype(np.int64) << 40)
            | (rec["j"].astype(np.int64) << 20) | rec["i"].astype(np.int64))


def _unpack(key):
    key = int(key)
    return (key >> 60, key & 0xFFFFF, (key >> 20) & 0xFFFFF, (key >> 40) & 0xFFFFF)


def _parent(keys):
    L = keys >> 60
    i, j, k = keys & 0xFFFFF, (keys >> 20) & 0xFFFFF, (keys >> 40) & 0xFFFFF
    return ((L - 1) << 60) | ((k >> 1) << 40) | ((j >> 1) << 20) | (i >> 1)


def near_mask(rec, alpha):
    """R19: a node is in the band if |U - alpha| <= 1e-6 (bound path) or, with a
    non-empty M~, |p1 - alpha| or |p2 - alpha| <= 1e-6."""
    U, p1, p2 = rec["U"], rec["p1"], rec["p2"]
    m = (np.abs(U - alpha) <= BAND) & (rec["ncase"] != 1)
    m |= (p1 >= 0) & ((np.abs(p1 - alpha) <= BAND) | (np.abs(p2 - alpha) <= BAND))
    return m


def excused_keys(keys, near_sorted, min_level=0):
    """True where the node or one of its ancestors (down to min_level) is in the band."""
    keys = np.asarray(keys, np.int64)
    out = np.zeros(len(keys), bool)
    cur = keys.copy()
    while len(cur):
        live = (cur >> 60) >= min_level
        if not live.any():
            break
        if len(near_sorted):
            pos = np.searchsorted(near_sorted, cur)
            hit = live & (pos < len(near_sorted)) & (near_sorted[np.minimum(pos, len(near_sorted) - 1)] == cur)
            out |= hit
        cur = np.where(live & ((cur >> 60) > 0), _parent(cur), -1)
        if np.all(cur < 0):
            break
    return out


def compare_node_sets(rec_g, rec_o, alpha, min_level=0):
    """C12 node-set comparison, vectorised.  A node evaluated on one side
    only, or with a different refine / case decision, is excused iff it or an ancestor
    (at level >= min_level) lies in the 1e-6 band on either side.
    Returns dict(unexcused, excused, common, max_dU, gpu_nodes, oracle_nodes, near)."""
    kg, ko = node_keys(rec_g), node_keys(rec_o)
    og, oo = np.argsort(kg, kind="stable"), np.argsort(ko, kind="stable")
    kg, ko = kg[og], ko[oo]
    assert len(np.unique(kg)) == len(kg) and len(np.unique(ko)) == len(ko), "duplicate node records"
    rg, ro = rec_g[og], rec_o[oo]
    near = np.unique(np.concatenate([kg[near_mask(rg, alpha)], ko[near_mask(ro, alpha)]]))
    only = np.setxor1d(kg, ko, assume_unique=True)
    common, ig, io = np.intersect1d(kg, ko, assume_unique=True, return_indices=True)
    gc, oc = rg[ig], ro[io]
    differ = (gc["refine"] != oc["refine"]) | (gc["ncase"] != oc["ncase"])
    ex_only = excused_keys(only, near, min_level)
    ex_diff = excused_keys(common[differ], near, min_level)
    unexcused = [_unpack(x) for x in np.concatenate([only[~ex_only], common[differ][~ex_diff]])]
    same = ~differ
    dU = np.abs(gc["U"][same].astype(np.float64) - oc["U"][same].astype(np.float64))
    return {"unexcused": unexcused, "excused": int(ex_only.sum() + ex_diff.sum()), "common": len(common),
            "max_dU": float(dU.max(initial=0.0)), "gpu_nodes": len(kg), "oracle_nodes": len(ko),
            "near": near}


def compare_leaf_sets(leaves_g, leaves_o, near, cells, lfull, max_depth, min_level=0):
    """Leaf cells present on one side only must lie under a band node (R19): each such
    cell's depth-max_depth node, or an ancestor, is in `near` (from compare_node_sets).
    Returns (n_only, n_unexcused)."""
    only = np.setxor1d(np.asarray(leaves_g, np.int64), np.asarray(leaves_o, np.int64))
    if len(only) == 0:
        return 0, 0
    nx, ny = cells[0], cells[1]
    x, y, z = only % nx, (only // nx) % ny, only // (nx * ny)
    s = lfull - max_depth
    keys = (np.int64(max_depth) << 60) | ((z >> s) << 40) | ((y >> s) << 20) | (x >> s)
    ex = excused_keys(keys, near, min_level)
    return len(only), int((~ex).sum())


def lcp_parity(lcp_g, lcp_o, N):
    d = np.abs(np.asarray(lcp_g, np.float64) - np.asarray(lcp_o, np.float64))
    frac_ok = float(np.mean(d <= 2.0 / N + 1e-7)) if len(d) else 1.0
    return frac_ok, float(d.mean()) if len(d) else 0.0, float(d.max(initial=0.0))
