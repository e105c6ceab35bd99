"""Host logic of the GPU-vs-oracle comparison (C12 node-set rule, R19): the vectorised
helpers in parity_util against a direct ancestor walk on perturbed oracle records."""
import numpy as np

import oracle as O
from parity_util import compare_leaf_sets, compare_node_sets, node_keys
from workloads import generate


def _records(name):
    w = generate(name)
    cfg = w.cfg
    M = O.Model.from_config(cfg, w.X, w.y)
    rec, leaves = M.octree(w.thetas[0], cfg.alpha, cfg.max_depth)
    return cfg, M, rec, leaves


def test_identical_sets_pass():
    cfg, M, rec, leaves = _records("t2")
    res = compare_node_sets(rec[::-1].copy(), rec, cfg.alpha)
    assert res["unexcused"] == [] and res["excused"] == 0 and res["common"] == len(rec)
    assert res["max_dU"] == 0.0
    assert compare_leaf_sets(leaves, leaves, res["near"], cfg.cells, M.lfull, cfg.max_depth) == (0, 0)


def test_flipped_decision_is_caught_unless_in_band():
    cfg, M, rec, leaves = _records("t2")
    g = np.random.default_rng(1)
    deep = np.nonzero((rec["level"] >= 3) & (rec["ncase"] != 1))[0]
    q = int(g.choice(deep))
    bad = rec.copy()
    bad["refine"][q] ^= 1
    res = compare_node_sets(bad, rec, cfg.alpha)
    key = tuple(int(rec[q][f]) for f in ("level", "i", "j", "k"))
    assert res["unexcused"] == [key]
    # put the node's ancestor two levels up into the band on the GPU side: excused
    L, i, j, k = key
    anc = np.nonzero((rec["level"] == L - 2) & (rec["i"] == i >> 2) & (rec["j"] == j >> 2)
                     & (rec["k"] == k >> 2))[0]
    assert len(anc) == 1
    bad["U"][anc[0]] = cfg.alpha + 0.5e-6
    bad["ncase"][anc[0]] = 0 if rec["ncase"][anc[0]] == 1 else bad["ncase"][anc[0]]
    res = compare_node_sets(bad, rec, cfg.alpha)
    assert res["unexcused"] == [] and res["excused"] >= 1
    # ... but not when the band node lies above min_level
    res = compare_node_sets(bad, rec, cfg.alpha, min_level=L - 1)
    assert res["unexcused"] == [key]


def test_missing_subtree_and_leaf_sets():
    cfg, M, rec, leaves = _records("t2")
    lf = M.lfull
    D = cfg.max_depth
    # drop one refined depth-(D-1) node's children (a missing subtree on the GPU side)
    par = np.nonzero((rec["level"] == D - 1) & (rec["refine"] == 1))[0][3]
    P = rec[par]
    kids = (rec["level"] == D) & (rec["i"] >> 1 == P["i"]) & (rec["j"] >> 1 == P["j"]) & (rec["k"] >> 1 == P["k"])
    assert kids.any()
    cut = rec[~kids]
    res = compare_node_sets(cut, rec, cfg.alpha)
    assert len(res["unexcused"]) == int(kids.sum())
    # the corresponding leaf cells differ and are unexcused
    s = lf - D
    nx, ny = cfg.cells[0], cfg.cells[1]
    x, y, z = leaves % nx, (leaves // nx) % ny, leaves // (nx * ny)
    under = ((x >> (s + 1)) == P["i"]) & ((y >> (s + 1)) == P["j"]) & ((z >> (s + 1)) == P["k"])
    n_only, n_unex = compare_leaf_sets(leaves[~under], leaves, res["near"], cfg.cells, lf, D)
    assert n_only == n_unex == int(under.sum()) > 0
    # with the parent in the band, everything below it is excused
    cut2 = cut.copy()
    q = np.nonzero(node_keys(cut2) == node_keys(rec[par:par + 1])[0])[0][0]
    cut2["p1"][q], cut2["p2"][q] = cfg.alpha, 0.7
    res = compare_node_sets(cut2, rec, cfg.alpha)
    assert res["unexcused"] == []
    assert compare_leaf_sets(leaves[~under], leaves, res["near"], cfg.cells, lf, D)[1] == 0
