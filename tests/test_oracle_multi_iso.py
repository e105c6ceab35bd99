"""Pins for the oracle's fused multi-isovalue leaf pass (NEXT-3, reading R27):
one sample stream per cell, the C11 crossing test applied to each of T
isovalues (the paper's isovalue sweep).  CPU only."""
import math

import numpy as np
from scipy import stats

import oracle as O
from workloads import generate


def test_multi_independent_corners_closed_form_every_theta():
    # diagonal Sigma: LCP(theta) = 1 - prod Phi((theta - mu)/sd) - prod (1 - Phi(...)) for
    # every theta of the sweep, all estimated from the same samples.
    g = np.random.default_rng(31)
    N = 40000
    thetas = np.array([-1.0, -0.5, -0.1, 0.0, 0.25, 0.6, 1.3])
    for trial in range(4):
        mu = g.normal(0, 0.6, 8)
        sd = g.uniform(0.3, 1.2, 8)
        got = O.mc_count_multi(mu, np.diag(sd), thetas, N, 500 + trial, trial, stream=3) / N
        for t, th in enumerate(thetas):
            p = stats.norm.cdf((th - mu) / sd)
            want = 1 - np.prod(p) - np.prod(1 - p)
            se = math.sqrt(max(want * (1 - want), 1e-12) / N)
            assert abs(got[t] - want) <= 4 * se + 1 / N, (trial, th, got[t], want)


def test_multi_is_the_single_pass_on_the_shared_stream():
    # R27: counts_multi[t] is exactly the single-isovalue count with counter word 3 = stream
    g = np.random.default_rng(32)
    A = g.standard_normal((8, 8)) * 0.3
    L = np.linalg.cholesky(A @ A.T + 0.1 * np.eye(8))
    mu = g.normal(0, 0.4, 8)
    thetas = np.array([-0.4, 0.0, 0.05, 0.7])
    got = O.mc_count_multi(mu, L, thetas, 3000, 9, 1234, stream=5)
    for t, th in enumerate(thetas):
        assert got[t] == O.mc_count(mu, L, th, 3000, 9, 1234, 5)
    # a different stream is a different sample set
    assert not np.array_equal(got, O.mc_count_multi(mu, L, thetas, 3000, 9, 1234, stream=6))


def test_multi_tails_and_point_mass():
    # thetas outside every sample's range never cross; a rank-0 posterior (L = 0) crosses
    # exactly the thetas equal to a corner value only when all corners coincide (ties cross, R24)
    mu = np.full(8, 0.25)
    assert O.mc_count_multi(mu, np.eye(8) * 0.1, [-50.0, 50.0], 2000, 1, 7).tolist() == [0, 0]
    got = O.mc_count_multi(mu, np.zeros((8, 8)), [0.0, 0.25, 0.5], 100, 1, 7)
    assert got.tolist() == [0, 100, 0]
    mu2 = np.array([0.0, 1, 0, 1, 0, 1, 0, 1], float)
    got = O.mc_count_multi(mu2, np.zeros((8, 8)), [-0.1, 0.0, 0.5, 1.0, 1.1], 10, 1, 7)
    assert got.tolist() == [0, 10, 10, 10, 0]


def test_pmc_cells_multi_mask_and_single_equivalence():
    w = generate("c1")
    M = O.Model.from_config(w.cfg, w.X, w.y)
    cells = np.array([0, 5, 77, 1000, 4095], np.int64)
    thetas = [-0.3, 0.0, 0.4]
    full = M.pmc_cells_multi(cells, thetas, 500, 17, stream=2)
    assert full.shape == (3, 5)
    for t, th in enumerate(thetas):
        np.testing.assert_array_equal(full[t], M.pmc_cells(cells, th, 500, 17, 2))
    mask = np.array([0b111, 0b001, 0b100, 0b000, 0b010], np.uint32)
    part = M.pmc_cells_multi(cells, thetas, 500, 17, stream=2, mask=mask)
    for t in range(3):
        on = (mask >> t) & 1 == 1
        np.testing.assert_array_equal(part[t][on], full[t][on])
        assert np.all(part[t][~on] == 0)
