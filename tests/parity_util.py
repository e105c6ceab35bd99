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


def _key(r):
    return (int(r["level"]), int(r["i"]), int(r["j"]), int(r["k"]))


def _near(r, alpha):
    if abs(r["U"] - alpha) <= BAND and r["ncase"] != 1:
        return True
    if r["p1"] >= 0 and (abs(r["p1"] - alpha) <= BAND or abs(r["p2"] - alpha) <= BAND):
        return True
    return False


def compare_node_sets(rec_g, rec_o, alpha):
    """C12 node-set comparison.  Returns dict(unexcused, excused, common, max_dU, case_mismatch)."""
    G = {_key(r): r for r in rec_g}
    O = {_key(r): r for r in rec_o}
    near = set(k for k, r in G.items() if _near(r, alpha)) | set(k for k, r in O.items() if _near(r, alpha))

    def excused(key):
        L, i, j, k = key
        while L >= 0:
            if (L, i, j, k) in near:
                return True
            L, i, j, k = L - 1, i // 2, j // 2, k // 2
        return False

    unexcused, excused_n = [], 0
    for key in set(G) ^ set(O):
        if excused(key):
            excused_n += 1
        else:
            unexcused.append(key)
    common = set(G) & set(O)
    max_dU = 0.0
    case_mm = 0
    for key in common:
        g, o = G[key], O[key]
        if g["refine"] != o["refine"] or g["ncase"] != o["ncase"]:
            if excused(key):
                excused_n += 1
                continue
            unexcused.append(key)
            case_mm += 1
            continue
        max_dU = max(max_dU, abs(float(g["U"]) - float(o["U"])))
    return {"unexcused": unexcused, "excused": excused_n, "common": len(common), "max_dU": max_dU,
            "gpu_nodes": len(G), "oracle_nodes": len(O)}


def lcp_parity(lcp_g, lcp_o, N):
    d = np.abs(np.asarray(lcp_g, np.float64) - np.asarray(lcp_o, np.float64))
    frac_ok = float(np.mean(d <= 2.0 / N + 1e-7)) if len(d) else 1.0
    return frac_ok, float(d.mean()) if len(d) else 0.0, float(d.max(initial=0.0))
