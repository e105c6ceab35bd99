"""Pins for the oracle's regional bound (C6) and octree (C7) (P7, P8)."""
import math

import numpy as np
import pytest
from scipy.special import ndtr

import oracle as O
from workloads import generate


def _model(name, **kw):
    w = generate(name)
    return w, O.Model.from_config(w.cfg, w.X, w.y, **kw)


def _vertex(cfg, i, j, k):
    h = [(cfg.hi[d] - cfg.lo[d]) / cfg.cells[d] for d in range(3)]
    return np.array([cfg.lo[0] + i * h[0], cfg.lo[1] + j * h[1], cfg.lo[2] + k * h[2]])


def _marg(M, cfg, i, j, k):
    mu, var = M.local_marginal(M.vertex_bucket(i, j, k), _vertex(cfg, i, j, k))
    return mu, math.sqrt(max(var, 1e-12 * cfg.variance))


def test_leaf_level_bound_closed_form():
    # h = 0 node (one cell, d = 8 corners): U = 1 - (min_c P(Y_c<th))^8 - (min_c P(Y_c>th))^8
    # (Eq. 4 with the exact discrete minimum of PAPER.md:158-166), one-sided in cases 2/3.
    w, M = _model("t1")
    cfg = w.cfg
    th, al = w.thetas[0], cfg.alpha
    L = M.lfull
    g = np.random.default_rng(0)
    checked = 0
    for _ in range(60):
        i, j, k = (int(g.integers(0, c)) for c in cfg.cells)
        rec = M.eval_node(th, al, L, i, j, k)
        if rec["ncase"] == 1:
            continue
        pl, ph = [], []
        for c in range(8):
            mu, sd = _marg(M, cfg, i + (c & 1), j + ((c >> 1) & 1), k + (c >> 2))
            pl.append(ndtr((th - mu) / sd))
            ph.append(ndtr((mu - th) / sd))
        bl, bu = min(pl), min(ph)
        want = {0: min(max(1 - bl ** 8 - bu ** 8, 0.0), 1.0), 2: 1 - bl ** 8, 3: 1 - bu ** 8}
        assert abs(rec["U"] - want[int(rec["ncase"])]) < 1e-12, (i, j, k, rec)
        checked += 1
    assert checked > 20


def test_node_records_bruteforce():
    # Alg. 1 lines 3-11 re-assembled in Python for random nodes of every level:
    # M~ by direct box test, candidate lattice by enumeration, bound by Eq. 4.
    for name in ("t1", "t2"):
        w, M = _model(name)
        cfg = w.cfg
        th, al = w.thetas[0], cfg.alpha
        h_cell = [(cfg.hi[d] - cfg.lo[d]) / cfg.cells[d] for d in range(3)]
        obs_cell = np.stack([np.clip(np.floor((w.X[:, d] - cfg.lo[d]) / h_cell[d]), 0,
                                     cfg.cells[d] - 1) for d in range(3)], 1).astype(int)
        g = np.random.default_rng(1)
        for level in range(0, cfg.max_depth + 1):
            hh = M.lfull - level
            side = 1 << hh
            n_ax = [-(-c // side) for c in cfg.cells]
            for _ in range(4):
                a = [int(g.integers(0, n)) for n in n_ax]
                rec = M.eval_node(th, al, level, *a)
                base = [a[d] * side for d in range(3)]
                vmax = [min(base[d] + side, cfg.cells[d]) for d in range(3)]
                inside = np.all((obs_cell >= base) & (obs_cell < np.array(base) + side), 1)
                if inside.any():
                    pl = []
                    for o in np.nonzero(inside)[0]:
                        mu, var = M.local_marginal(M.point_bucket(w.X[o]), w.X[o])
                        sd = math.sqrt(max(var, 1e-12 * cfg.variance))
                        pl.append(ndtr((th - mu) / sd))
                    p1, p2 = max(pl), max(1 - p for p in pl)
                    assert abs(rec["p1"] - p1) < 1e-12 and abs(rec["p2"] - p2) < 1e-9
                else:
                    assert rec["p1"] == -1 and rec["p2"] == -1
                    p1 = p2 = -1
                if inside.any() and p1 > al and p2 > al:
                    assert rec["ncase"] == 1 and rec["refine"] == 1
                    continue
                stride = 1 << max(0, hh - cfg.h_full)
                axes = [sorted(set(list(range(base[d], vmax[d], stride)) + [vmax[d]])) for d in range(3)]
                qlo = qhi = 0.0
                for vk in axes[2]:
                    for vj in axes[1]:
                        for vi in axes[0]:
                            mu, sd = _marg(M, cfg, vi, vj, vk)
                            qlo = max(qlo, ndtr((mu - th) / sd))
                            qhi = max(qhi, ndtr((th - mu) / sd))
                d = np.prod([vmax[q] - base[q] + 1 for q in range(3)])
                ncase = 0 if not inside.any() else (2 if p2 <= al else 3)
                assert rec["ncase"] == ncase
                if ncase == 2:
                    U = -_expm1(d * _l1m(qlo))
                elif ncase == 3:
                    U = -_expm1(d * _l1m(qhi))
                else:
                    U = min(max(-_expm1(d * _l1m(qlo)) - _exp(d * _l1m(qhi)), 0), 1)
                assert abs(rec["U"] - U) <= 1e-9 * max(U, 1e-300) + 1e-15, (name, level, a, rec["U"], U)
                assert rec["refine"] == (rec["U"] > al)


def _expm1(x):
    return -1.0 if x == -math.inf else math.expm1(x)


def _exp(x):
    return 0.0 if x == -math.inf else math.exp(x)


def _l1m(q):
    return -math.inf if q >= 1.0 else math.log1p(-q)


def _cells_of(cfg, lfull, level, i, j, k):
    side = 1 << (lfull - level)
    out = []
    for z in range(k * side, min((k + 1) * side, cfg.cells[2])):
        for y in range(j * side, min((j + 1) * side, cfg.cells[1])):
            for x in range(i * side, min((i + 1) * side, cfg.cells[0])):
                out.append(x + cfg.cells[0] * (y + cfg.cells[1] * z))
    return out


@pytest.mark.parametrize("name", ["c1", "t1", "t2"])
def test_octree_partition_and_cases(name):
    # every cell is finalised exactly once; children tile parents;
    # case exclusivity; leaves = cells of refined depth-D nodes.
    w, M = _model(name)
    cfg = w.cfg
    recs, leaves = M.octree(w.thetas[0], cfg.alpha, cfg.max_depth)
    lf = M.lfull
    total = cfg.cells[0] * cfg.cells[1] * cfg.cells[2]
    final = np.zeros(total, int)
    by_key = {(int(r["level"]), int(r["i"]), int(r["j"]), int(r["k"])): r for r in recs}
    assert len(by_key) == len(recs)
    for r in recs:
        key = (int(r["level"]), int(r["i"]), int(r["j"]), int(r["k"]))
        if key[0] > 0:
            parent = (key[0] - 1, key[1] // 2, key[2] // 2, key[3] // 2)
            assert by_key[parent]["refine"] == 1
        if r["p1"] >= 0:
            assert not (r["p1"] <= cfg.alpha and r["p2"] <= cfg.alpha)
            assert (r["ncase"] == 1) == (r["p1"] > cfg.alpha and r["p2"] > cfg.alpha)
        else:
            assert r["ncase"] == 0
        assert 0.0 <= r["U"] <= 1.0
        if not r["refine"] or key[0] == cfg.max_depth:
            final[_cells_of(cfg, lf, *key)] += 1
        if r["refine"] and key[0] < cfg.max_depth:
            kids = [(key[0] + 1, 2 * key[1] + (c & 1), 2 * key[2] + ((c >> 1) & 1), 2 * key[3] + (c >> 2))
                    for c in range(8)]
            kids = [c for c in kids if _cells_of(cfg, lf, *c)]
            assert all(c in by_key for c in kids)
    assert np.all(final == 1)
    want = sorted(c for r in recs if r["refine"] and r["level"] == cfg.max_depth
                  for c in _cells_of(cfg, lf, int(r["level"]), int(r["i"]), int(r["j"]), int(r["k"])))
    assert np.array_equal(leaves, np.array(want, dtype=np.int64))


def test_alpha_to_zero_refines_everything():
    # alpha -> 0+: every node refines, so the leaf set is the whole grid and the
    # pruned LCP field equals the dense baseline bit for bit.
    w, M = _model("t2")
    cfg = w.cfg
    recs, leaves = M.octree(w.thetas[0], 1e-300, cfg.max_depth)
    total = cfg.cells[0] * cfg.cells[1] * cfg.cells[2]
    assert np.array_equal(leaves, np.arange(total))
    sub = leaves[::97]
    a = M.pmc_cells(sub, w.thetas[0], 200, 5)
    b = M.pmc_cells(np.arange(total)[::97], w.thetas[0], 200, 5)
    assert np.array_equal(a, b)


def test_far_shifted_field_prunes_root():
    # mean >= theta + 10 sigma everywhere: empty leaf set, root pruned
    w = generate("t1")
    cfg = w.cfg
    M = O.Model.from_config(cfg, w.X, w.y)
    recs, leaves = M.octree(-25.0, cfg.alpha, cfg.max_depth)
    assert len(leaves) == 0 and len(recs) == 1 and recs[0]["refine"] == 0
    recs, leaves = M.octree(+25.0, cfg.alpha, cfg.max_depth)
    assert len(leaves) == 0 and len(recs) == 1


def test_bound_soundness_c1_bruteforce():
    # BASELINE pin: on the tiny grid (h_full = D, exact discrete minimum) the
    # bound U of a node is >= the brute-force MC LCP of every cell it covers,
    # up to 3 SE; Slepian needs non-negative correlations (R12) so violations are
    # counted and must stay <= 0.5 %.
    w, M = _model("c1")
    cfg = w.cfg
    th = w.thetas[0]
    # a larger alpha makes more nodes informative (pruned / near-pruned)
    recs, _ = M.octree(th, 0.05, cfg.max_depth)
    N = 20000
    lf = M.lfull
    pairs = []
    for r in recs:
        if r["ncase"] == 1 or r["U"] > 0.2:
            continue
        for c in _cells_of(cfg, lf, int(r["level"]), int(r["i"]), int(r["j"]), int(r["k"])):
            pairs.append((c, r["U"]))
    assert len(pairs) > 50
    cells = np.array([p[0] for p in pairs], np.int64)
    U = np.array([p[1] for p in pairs])
    lcp = M.pmc_cells(cells, th, N, 12345)
    se = np.sqrt(np.maximum(lcp * (1 - lcp), 1.0 / N) / N)
    viol = lcp > U + 3 * se + 1.0 / N
    assert viol.mean() <= 0.005, (viol.sum(), len(pairs))
