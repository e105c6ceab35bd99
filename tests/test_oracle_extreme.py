"""Pins for NEXT-1 (R26): the continuous extreme search of the regional bound
(PAPER.md:172 any point of the region; :183 quasi-Newton search with a closed-
form gradient).  CPU only."""
import math

import numpy as np
import pytest

import oracle as O
from workloads import generate


def _model(name):
    w = generate(name)
    return w, O.Model.from_config(w.cfg, w.X, w.y)


@pytest.mark.parametrize("name", ["t1", "t2", "c1"])
def test_f_gradient_matches_finite_differences(name):
    w, M = _model(name)
    cfg = w.cfg
    g = np.random.default_rng(3)
    th = w.thetas[0]
    for _ in range(25):
        x = np.asarray(cfg.lo) + (np.asarray(cfg.hi) - np.asarray(cfg.lo)) * g.random(3)
        b = M.point_bucket(x)
        f, grad = M.f_grad(b, x, th)
        mu, var = M.local_marginal(b, x)
        assert abs(f - (mu - th) / (math.sqrt(max(var, 1e-12 * cfg.variance)) * math.sqrt(2))) < 1e-12 * max(1, abs(f))
        eps = 1e-6 * min(cfg.lengthscale)
        for d in range(3):
            e = np.zeros(3)
            e[d] = eps
            fd = (M.f_grad(b, x + e, th)[0] - M.f_grad(b, x - e, th)[0]) / (2 * eps)
            assert abs(fd - grad[d]) <= 1e-5 * max(1.0, abs(grad[d])), (d, fd, grad[d])


@pytest.mark.parametrize("name", ["t1", "c2"])
def test_search_improves_on_lattice_and_matches_scan(name):
    # the search starts at the lattice extreme and only accepts improvements;
    # a dense 13^3 scan of f over the node box (same local model) bounds how
    # much it can miss (a local optimum: allowed, but rare).
    w, M = _model(name)
    cfg = w.cfg
    th = w.thetas[0]
    M.set_extreme(48)
    lf = M.lfull
    h = [(cfg.hi[d] - cfg.lo[d]) / cfg.cells[d] for d in range(3)]
    rng = np.random.default_rng(5)
    close = tot = 0
    for level in range(1, lf - cfg.h_full):
        hh = lf - level
        side = 1 << hh
        n_ax = [-(-c // side) for c in cfg.cells]
        for _ in range(6):
            a = [int(rng.integers(0, n)) for n in n_ax]
            zl_max, zl_min, zs_max, zs_min, f0_max, f0_min = M.node_extremes(th, level, *a)
            # monotone: the search only accepts improvements over its start (the lattice
            # extreme vertex, evaluated with the search's local model)
            assert zs_max >= f0_max and zs_min <= f0_min
            base = [a[d] * side for d in range(3)]
            vmax = [min(base[d] + side, cfg.cells[d]) for d in range(3)]
            if level < cfg.bucket_log2:
                continue
            b = M.vertex_bucket(*base)
            ts = np.linspace(0, 1, 13)
            best = -np.inf
            for tz in ts:
                for ty in ts:
                    for tx in ts:
                        x = [cfg.lo[d] + (base[d] + t * (vmax[d] - base[d])) * h[d] for d, t in enumerate((tx, ty, tz))]
                        best = max(best, M.f_grad(b, x, th)[0])
            tot += 1
            close += zs_max >= best - 1e-3 * max(1.0, abs(best))
    assert tot > 0 and close / tot >= 0.75, (close, tot)


def test_search_only_loosens_the_bound():
    # U with the continuous search >= U with the lattice alone (Q can only grow),
    # so every node the lattice run refines is refined again.
    w, M = _model("c2")
    cfg = w.cfg
    th = w.thetas[0]
    rec_l, leaves_l = M.octree(th, cfg.alpha, cfg.max_depth)
    M.set_extreme(16)
    rec_e, leaves_e = M.octree(th, cfg.alpha, cfg.max_depth)
    E = {(int(r["level"]), int(r["i"]), int(r["j"]), int(r["k"])): r for r in rec_e}
    for r in rec_l:
        key = (int(r["level"]), int(r["i"]), int(r["j"]), int(r["k"]))
        assert key in E
        assert E[key]["U"] >= r["U"] - 1e-15
        assert E[key]["refine"] >= r["refine"]
    assert set(leaves_l.tolist()) <= set(leaves_e.tolist())


@pytest.mark.parametrize("name", ["t1", "t2", "c2"])
def test_search_matches_scipy_lbfgsb(name):
    # R26b against scipy's L-BFGS-B (PAPER.md:183 names the method) on the same objective,
    # box and start: maximise f = (mu - theta) / (sigma sqrt 2) of the node's local model over
    # the node box (and minimise it), from the lattice extreme.  Both are local quasi-Newton
    # searches with a closed-form gradient; they agree on >= 95 % of the nodes to 1e-6.
    from scipy.optimize import minimize
    w, M = _model(name)
    cfg = w.cfg
    th = w.thetas[0]
    M.set_extreme(64)
    lf = M.lfull
    h = [(cfg.hi[d] - cfg.lo[d]) / cfg.cells[d] for d in range(3)]
    rng = np.random.default_rng(11)
    agree = not_worse = tot = 0
    worst = []
    for level in range(max(1, cfg.bucket_log2), lf - cfg.h_full):
        side = 1 << (lf - level)
        n_ax = [-(-c // side) for c in cfg.cells]
        for _ in range(12):
            a = [int(rng.integers(0, n)) for n in n_ax]
            ext, x_max, x_min = M.node_extremes(th, level, *a, starts=True)
            base = [a[d] * side for d in range(3)]
            vmax = [min(base[d] + side, cfg.cells[d]) for d in range(3)]
            b = M.vertex_bucket(*base)
            bounds = [(cfg.lo[d] + base[d] * h[d], cfg.lo[d] + vmax[d] * h[d]) for d in range(3)]
            for sgn, x0, got in ((1.0, x_max, ext[2]), (-1.0, x_min, ext[3])):
                def phi(x, sgn=sgn):
                    f, gr = M.f_grad(b, x, th)
                    return -sgn * f, -sgn * np.asarray(gr)
                r = minimize(phi, x0, jac=True, method="L-BFGS-B", bounds=bounds,
                             options={"maxiter": 500, "gtol": 1e-12, "ftol": 1e-15})
                ref = -sgn * r.fun
                tot += 1
                tol = 1e-6 * max(1.0, abs(ref))
                agree += abs(got - ref) <= tol
                not_worse += sgn * (got - ref) >= -tol     # a better local optimum is allowed
                if abs(got - ref) > tol:
                    worst.append((level, a, sgn, got, ref))
    print(f"{name}: {agree}/{tot} within 1e-6 of scipy L-BFGS-B, {not_worse}/{tot} at least as good", worst[:4])
    assert tot >= 24 and not_worse / tot >= 0.95 and agree / tot >= 0.9, (agree, not_worse, tot, worst[:5])
