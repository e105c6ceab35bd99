"""Pins for the oracle's beta-box local sets (NEXT-2, reading R28):
bucket b's local GP uses every observation inside the bucket box enlarged by
beta * l_d per axis.  CPU only."""
import numpy as np
import pytest
from scipy.linalg import cho_factor, cho_solve

import oracle as O


def _setup(seed=3, m=80, cells=(12, 10, 8), ls=(0.12, 0.15, 0.1)):
    g = np.random.default_rng(seed)
    lo, hi = np.zeros(3), np.array([1.0, 0.9, 0.7])
    X = lo + (hi - lo) * g.random((m, 3))
    y = np.sin(4 * X[:, 0]) + X[:, 1] - X[:, 2] ** 2 + 0.01 * g.standard_normal(m)
    kern = O.make_kernel(0, 1.0, ls, 1e-4, 0.1)
    grid = O.make_grid(lo, hi, cells)
    return kern, grid, X, y, np.asarray(ls), lo, hi, np.asarray(cells)


def _box_members(X, lo, h, bs, bi, beta, ls):
    # the same bounds evaluated independently in numpy (left to right, no FMA)
    blo = (lo + (bi * bs) * h) - beta * ls
    bhi = (lo + ((bi + 1) * bs) * h) + beta * ls
    return np.nonzero(np.all((X >= blo) & (X < bhi), axis=1))[0]


@pytest.mark.parametrize("beta", [0.5, 1.0, 2.0])
def test_box_sets_match_brute_force(beta):
    kern, grid, X, y, ls, lo, hi, cells = _setup()
    M = O.Model.box(kern, grid, X, y, len(X), 2, 2, beta)
    lf = M.lfull
    bs = 1 << (lf - 2)
    h = (hi - lo) / cells
    nb = (cells + bs - 1) // bs
    for b in range(M.nbuckets):
        bi = np.array([b % nb[0], (b // nb[0]) % nb[1], b // (nb[0] * nb[1])])
        want = _box_members(X, lo, h, bs, bi, beta, ls)
        got = M.bucket_set(b)
        np.testing.assert_array_equal(got[: len(want)], want)
        assert np.all(got[len(want):] == -1)


def test_box_local_marginal_is_exact_gp_on_the_box_set():
    # library pin: the local posterior equals scipy's Cholesky solve on the box subset
    kern, grid, X, y, ls, lo, hi, cells = _setup()
    M = O.Model.box(kern, grid, X, y, len(X), 2, 2, 1.0)
    g = np.random.default_rng(1)
    for _ in range(20):
        x = lo + (hi - lo) * g.random(3)
        b = M.point_bucket(x)
        S = M.bucket_set(b)
        S = S[S >= 0]
        mu, var = M.local_marginal(b, x)
        if len(S) == 0:
            assert abs(mu - 0.1) < 1e-15 and abs(var - 1.0) < 1e-15
            continue
        d = (X[S][:, None, :] - X[S][None, :, :]) / ls
        K = np.exp(-0.5 * (d ** 2).sum(-1)) + 1e-4 * np.eye(len(S))
        kx = np.exp(-0.5 * (((X[S] - x) / ls) ** 2).sum(-1))
        cf = cho_factor(K, lower=True)
        assert abs(mu - (0.1 + kx @ cho_solve(cf, y[S] - 0.1))) < 1e-10
        assert abs(var - (1.0 - kx @ cho_solve(cf, kx))) < 1e-10


def test_box_covering_everything_is_the_exact_gp():
    # beta large enough that every box holds all m observations: k = m exact GP (C2)
    kern, grid, X, y, ls, lo, hi, cells = _setup(m=40)
    M = O.Model.box(kern, grid, X, y, len(X), 2, 2, 20.0)
    g = np.random.default_rng(2)
    Q = lo + (hi - lo) * g.random((10, 3))
    mu_e, cov_e = O.gp_exact(kern, X, y, Q)
    for q in range(len(Q)):
        mu, var = M.local_marginal(M.point_bucket(Q[q]), Q[q])
        assert abs(mu - mu_e[q]) < 1e-10 and abs(var - cov_e[q, q]) < 1e-10


def test_box_larger_than_k_is_an_error():
    kern, grid, X, y, ls, lo, hi, cells = _setup()
    with pytest.raises(O.OracleError):
        O.Model.box(kern, grid, X, y, 5, 2, 2, 1.0)
