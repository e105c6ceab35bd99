"""Pins for the oracle's kernel, exact GP and local GP (P1-P4).

Each check compares the oracle with something it does not compute itself:
closed forms, special cases the paper fixes, the paper's own Eq. 1 form, or
brute force.  CPU only.
"""
import math

import numpy as np
import pytest

import oracle as O
from workloads import generate, get_config


SE, MAT = 0, 1


def rng(seed=0):
    return np.random.default_rng(seed)


# ----------------------------------------------------------------- P1 kernel
def test_kernel_closed_forms():
    kse = O.make_kernel(SE, 2.5, 0.3, 0.0)
    kma = O.make_kernel(MAT, 1.7, 0.4, 0.0)
    x = np.array([0.1, 0.2, 0.3])
    assert O.kernel_value(kse, x, x) == 2.5
    assert O.kernel_value(kma, x, x) == 1.7
    # SE at distance l sqrt(2 ln 2) is sigma^2 / 2
    r = 0.3 * math.sqrt(2 * math.log(2))
    assert abs(O.kernel_value(kse, x, x + np.array([r, 0, 0])) - 1.25) < 1e-14
    # Matern-5/2 at r = l: (1 + sqrt5 + 5/3) e^-sqrt5
    want = 1.7 * (1 + math.sqrt(5) + 5 / 3) * math.exp(-math.sqrt(5))
    assert abs(O.kernel_value(kma, x, x + np.array([0, 0.4, 0])) - want) < 1e-14
    # anisotropic SE: each axis scaled by its own length
    kan = O.make_kernel(SE, 1.0, (0.1, 0.2, 0.4), 0.0)
    d = np.array([0.1, 0.2, 0.4])
    assert abs(O.kernel_value(kan, x, x + d) - math.exp(-1.5)) < 1e-15


def test_kernel_symmetry_and_psd():
    g = rng(1)
    P = g.random((30, 3))
    for kern in (O.make_kernel(SE, 1.0, 0.2, 0.0), O.make_kernel(MAT, 1.0, (0.1, 0.2, 0.3), 0.0)):
        K = np.array([[O.kernel_value(kern, a, b) for b in P] for a in P])
        assert np.array_equal(K, K.T)
        assert np.linalg.eigvalsh(K).min() > -1e-12


# -------------------------------------------------------------- P2 exact GP
def test_single_observation_closed_form():
    # m = 1: mu(q) = m0 + k(q,x)(y - m0)/(s^2 + sn^2), var = s^2 - k(q,x)^2/(s^2 + sn^2)
    kern = O.make_kernel(SE, 1.3, 0.25, 0.01, prior_mean=0.2)
    X = np.array([[0.5, 0.5, 0.5]])
    y = np.array([1.1])
    Q = np.array([[0.6, 0.45, 0.5], [0.9, 0.1, 0.2]])
    mu, cov = O.gp_exact(kern, X, y, Q)
    for q in range(2):
        kq = O.kernel_value(kern, Q[q], X[0])
        assert abs(mu[q] - (0.2 + kq * 0.9 / 1.31)) < 1e-14
        assert abs(cov[q, q] - (1.3 - kq * kq / 1.31)) < 1e-14
    k01 = O.kernel_value(kern, Q[0], Q[1])
    kq0, kq1 = O.kernel_value(kern, Q[0], X[0]), O.kernel_value(kern, Q[1], X[0])
    assert abs(cov[0, 1] - (k01 - kq0 * kq1 / 1.31)) < 1e-14


def test_zero_noise_interpolates():
    # BASELINE north_star pin: the zero-noise posterior interpolates the
    # observations with zero variance.
    g = rng(2)
    X = g.random((15, 3))
    y = g.standard_normal(15)
    for kind in (SE, MAT):
        kern = O.make_kernel(kind, 1.0, 0.15, 0.0)
        mu, cov = O.gp_exact(kern, X, y, X)
        assert np.abs(mu - y).max() < 1e-8
        assert np.abs(np.diag(cov)).max() < 1e-8


def test_far_field_is_prior():
    g = rng(3)
    X = g.random((20, 3))
    y = g.standard_normal(20)
    kern = O.make_kernel(SE, 0.7, 0.05, 1e-4, prior_mean=-0.3)
    mu, cov = O.gp_exact(kern, X, y, np.array([[50.0, 50.0, 50.0], [60.0, -40.0, 5.0]]))
    assert np.allclose(mu, -0.3, atol=1e-14)
    assert np.allclose(np.diag(cov), 0.7, atol=1e-14)
    assert abs(cov[0, 1]) < 1e-14


def test_eq1_sgpr_identity():
    # PAPER.md:89-95, Eq. 1 with M = X, mu_M = K (K + sn^2 I)^-1 y and
    # A_M = sn^2 K (K + sn^2 I)^-1 must equal the oracle's GP regression form (R1).
    g = rng(4)
    X = g.random((25, 3))
    y = g.standard_normal(25)
    Q = g.random((6, 3))
    sn2 = 3e-3
    kern = O.make_kernel(SE, 1.0, 0.3, sn2)
    K = np.array([[O.kernel_value(kern, a, b) for b in X] for a in X])
    KQX = np.array([[O.kernel_value(kern, a, b) for b in X] for a in Q])
    KQQ = np.array([[O.kernel_value(kern, a, b) for b in Q] for a in Q])
    Ky = K + sn2 * np.eye(25)
    muM = K @ np.linalg.solve(Ky, y)
    AM = sn2 * K @ np.linalg.inv(Ky)
    Kinv = np.linalg.inv(K)
    mu_eq1 = KQX @ Kinv @ muM
    S_eq1 = KQQ - KQX @ Kinv @ KQX.T + KQX @ Kinv @ AM @ Kinv @ KQX.T
    mu, cov = O.gp_exact(kern, X, y, Q)
    assert np.abs(mu - mu_eq1).max() < 1e-7
    assert np.abs(cov - S_eq1).max() < 1e-7


def test_marginalisation_consistency():
    g = rng(5)
    X = g.random((30, 3))
    y = g.standard_normal(30)
    kern = O.make_kernel(MAT, 1.0, 0.2, 1e-4)
    Q = g.random((8, 3))
    mu, cov = O.gp_exact(kern, X, y, Q)
    for q in (0, 3, 7):
        m1, c1 = O.gp_exact(kern, X, y, Q[q:q + 1])
        assert abs(m1[0] - mu[q]) < 1e-13 and abs(c1[0, 0] - cov[q, q]) < 1e-13
    assert np.allclose(cov, cov.T, atol=1e-15)
    assert np.linalg.eigvalsh(cov).min() > -1e-10


# ---------------------------------------------------------- P3 local GP
def _model(name, **kw):
    w = generate(name)
    return w, O.Model.from_config(w.cfg, w.X, w.y, **kw)


def test_knn_bruteforce():
    # S_B = k smallest sum_d ((x_d - c_d) / l_d)^2, ties to the lower index (R2):
    # independent numpy lexsort over all observations.
    for name in ("t1", "t2", "c2"):
        w, M = _model(name)
        cfg = w.cfg
        lf = M.lfull
        bs = 1 << (lf - cfg.bucket_log2)
        nb = [-(-c // bs) for c in cfg.cells]
        h = [(cfg.hi[d] - cfg.lo[d]) / cfg.cells[d] for d in range(3)]
        wgt = [1.0 / l for l in cfg.lengthscale]
        for b in range(M.nbuckets):
            bi = (b % nb[0], (b // nb[0]) % nb[1], b // (nb[0] * nb[1]))
            c = [cfg.lo[d] + (bi[d] + 0.5) * (bs * h[d]) for d in range(3)]
            t = [(w.X[:, d] - c[d]) * wgt[d] for d in range(3)]
            d2 = t[0] * t[0] + t[1] * t[1] + t[2] * t[2]
            order = np.lexsort((np.arange(len(d2)), d2))
            assert np.array_equal(np.sort(order[:cfg.k]), M.bucket_set(b)), (name, b)


def test_point_and_vertex_buckets():
    w, M = _model("t2")
    cfg = w.cfg
    lf = M.lfull
    bs = 1 << (lf - cfg.bucket_log2)
    nb = [-(-c // bs) for c in cfg.cells]
    h = [(cfg.hi[d] - cfg.lo[d]) / cfg.cells[d] for d in range(3)]
    g = rng(6)
    pts = np.asarray(cfg.lo) + (np.asarray(cfg.hi) - np.asarray(cfg.lo)) * g.random((200, 3))
    pts[:5] = cfg.hi  # the far faces clamp into the last bucket
    for p in pts:
        idx = [min(max(int(math.floor((p[d] - cfg.lo[d]) / (bs * h[d]))), 0), nb[d] - 1)
               for d in range(3)]
        assert M.point_bucket(p) == idx[0] + nb[0] * (idx[1] + nb[1] * idx[2])
    nx, ny, nz = cfg.cells
    assert M.vertex_bucket(nx, ny, nz) == M.nbuckets - 1
    for cell in (0, 7, nx * ny * nz - 1, 1234):
        i, j, k = cell % nx, (cell // nx) % ny, cell // (nx * ny)
        assert M.cell_bucket(cell) == (i // bs) + nb[0] * ((j // bs) + nb[1] * (k // bs))


def test_local_gp_with_k_equal_m_is_exact_gp():
    # BASELINE north_star pin: the local GP with k = m equals the global GP.
    for name in ("c1", "t1"):
        w = generate(name)
        cfg = w.cfg
        M = O.Model.from_config(cfg, w.X, w.y, k=cfg.m)
        kern = O.make_kernel(cfg.kernel, cfg.variance, cfg.lengthscale, cfg.nugget, cfg.prior_mean)
        nx, ny, nz = cfg.cells
        h = [(cfg.hi[d] - cfg.lo[d]) / cfg.cells[d] for d in range(3)]
        for cell in (0, 17, nx * ny * nz // 2 + 3, nx * ny * nz - 1):
            i, j, k = cell % nx, (cell // nx) % ny, cell // (nx * ny)
            Q = np.array([[cfg.lo[0] + (i + (c & 1)) * h[0], cfg.lo[1] + (j + ((c >> 1) & 1)) * h[1],
                           cfg.lo[2] + (k + (c >> 2)) * h[2]] for c in range(8)])
            mu_e, cov_e = O.gp_exact(kern, w.X, w.y, Q)
            mu_l, cov_l = M.cell_posterior(cell)
            assert np.abs(mu_l - mu_e).max() < 1e-11
            assert np.abs(cov_l - cov_e).max() < 1e-11
            b = M.cell_bucket(cell)
            m1, v1 = M.local_marginal(b, Q[5])
            assert abs(m1 - mu_e[5]) < 1e-11 and abs(v1 - cov_e[5, 5]) < 1e-11


def test_local_marginal_matches_cell_posterior_diagonal():
    w, M = _model("t2")
    for cell in (0, 100, 5000, 11879):
        mu, cov = M.cell_posterior(cell)
        b = M.cell_bucket(cell)
        cfg = w.cfg
        nx, ny = cfg.cells[0], cfg.cells[1]
        i, j, k = cell % nx, (cell // nx) % ny, cell // (nx * ny)
        h = [(cfg.hi[d] - cfg.lo[d]) / cfg.cells[d] for d in range(3)]
        x7 = [cfg.lo[0] + (i + 1) * h[0], cfg.lo[1] + (j + 1) * h[1], cfg.lo[2] + (k + 1) * h[2]]
        m, v = M.local_marginal(b, x7)
        assert abs(m - mu[7]) < 1e-13 and abs(v - cov[7, 7]) < 1e-13


# ------------------------------------------------------------------ P4 Phi
def _golden(name):
    import os
    rows = []
    for line in open(os.path.join(os.path.dirname(__file__), "golden", name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append(line.split())
    return rows


def test_phi_golden():
    for z, phi in _golden("normal_cdf.txt"):
        z, phi = float(z), float(phi)
        # P(Y < theta) with Y ~ N(mu, var): z = (theta - mu) / sigma
        plo, phi_ = O.tail_probs(0.3, 4.0, 0.3 + 2.0 * z)
        assert abs(plo - phi) <= 1e-13 * max(phi, 1e-300) + 1e-16, (z, plo, phi)
        assert abs(phi_ - (1.0 - phi)) < 1e-15 or abs(phi_ / (1.0 - phi) - 1) < 1e-13


def test_phi_tails_relative_precision():
    # erfc keeps the small tail exact; P< + P> = 1
    for z in np.linspace(-30, 30, 61):
        a, b = O.tail_probs(0.0, 1.0, float(z))
        assert abs(a + b - 1.0) < 2e-16 * 4
        assert a > 0 and b > 0 or abs(z) > 37
