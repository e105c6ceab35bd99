"""Pins for the oracle's Philox RNG, normals, 8x8 Cholesky and MC estimator
(P5, P6, P9).  CPU only."""
import math
import os
import shutil
import subprocess

import numpy as np
import pytest
from scipy import stats

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


def _golden(name):
    rows = []
    for line in open(os.path.join(HERE, "golden", name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append(line.split())
    return rows


# ----------------------------------------------------------------- P6 Philox
def test_philox_published_kat():
    for row in _golden("philox4x32_10_kat.txt"):
        v = [int(t, 16) for t in row]
        out = O.philox4x32_10(v[0:4], v[4:6])
        assert out.tolist() == v[6:10]


CURAND_KAT_SRC = r"""
#define QUALIFIERS static __forceinline__ __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>
int main() {
  unsigned s = 12345u;
  for (int t = 0; t < 200; ++t) {
    unsigned v[6];
    for (int q = 0; q < 6; ++q) { s = s * 1664525u + 1013904223u; v[q] = s; }
    uint4 c = make_uint4(v[0], v[1], v[2], v[3]); uint2 k = make_uint2(v[4], v[5]);
    uint4 r = curand_Philox4x32_10(c, k);
    printf("%u %u %u %u %u %u %u %u %u %u\n", v[0], v[1], v[2], v[3], v[4], v[5], r.x, r.y, r.z, r.w);
  }
}
"""


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_philox_vs_curand_host(tmp_path):
    # Library pin: CUDA's own curand_Philox4x32_10, compiled for the host.
    src = tmp_path / "kat.cu"
    src.write_text(CURAND_KAT_SRC)
    exe = tmp_path / "kat"
    subprocess.check_call(["nvcc", "-Wno-deprecated-gpu-targets", "-o", str(exe), str(src)])
    out = subprocess.check_output([str(exe)]).decode().split("\n")
    n = 0
    for line in out:
        if not line.strip():
            continue
        v = [int(t) for t in line.split()]
        assert O.philox4x32_10(v[0:4], v[4:6]).tolist() == v[6:10]
        n += 1
    assert n == 200


def _bm(ra, rb):
    ua, ub = [((int(x) & 0x7FFFFF) + 0.5) / 2 ** 23 for x in (ra, rb)]
    R = math.sqrt(-2 * math.log(ua))
    return R * math.cos(2 * math.pi * ub), R * math.sin(2 * math.pi * ub)


@pytest.mark.parametrize("s", [0, 5, 37, 70, 101, 127, 128, 300, 4095])
def test_normals_layout_and_uniform_map(s):
    # DESIGN R13 / R13c, written out from the text: key = (seed lo, seed hi); u from the low 23
    # bits.  z0..z3: group g = 32 (s div 128) + s mod 32, position t = (s div 32) mod 4; the
    # group's word stream = the 12 words of the blocks with counter word 3 = 2 (3g + j), j < 3;
    # the sample takes stream words 3t..3t+2 = (A, B, C): (z0, z1) = BM(A, C),
    # (z2, z3) = BM(B, top bytes of A, B, C).  z4..z7: block 2s + 1, pairs (0, 1), (2, 3).
    seed, cell, iso = 0x1234567890ABCDEF, (7 << 32) + 99, 2
    z = O.normals8(seed, cell, iso, s)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    ctr = lambda w: [cell & 0xFFFFFFFF, iso, cell >> 32, w]
    g, t = 32 * (s // 128) + s % 32, (s // 32) % 4
    stream = [int(x) for j in range(3) for x in O.philox4x32_10(ctr(2 * (3 * g + j)), key)]
    A, B, C = stream[3 * t:3 * t + 3]
    D = (A >> 24) | ((B >> 24) << 8) | ((C >> 24) << 16)
    r = [int(x) for x in O.philox4x32_10(ctr(2 * s + 1), key)]
    want = [*_bm(A, C), *_bm(B, D), *_bm(r[0], r[1]), *_bm(r[2], r[3])]
    assert np.abs(np.asarray(z) - np.asarray(want)).max() < 1e-15


def test_normals_words_not_shared():
    # every phase-1 word of a 128-sample block of a lane group is used by exactly one sample,
    # and no counter of phase 1 (even) meets one of phase 2 (odd)
    seen = {}
    for s in range(1024):
        g, t = 32 * (s // 128) + s % 32, (s // 32) % 4
        for i in range(3 * t, 3 * t + 3):
            w = (2 * (3 * g + i // 4), i % 4)
            assert w not in seen, (s, seen.get(w))
            seen[w] = s
    assert len(seen) == 3 * 1024 and all(w % 2 == 0 for w, _ in seen)


def test_normals_statistics():
    # 8 x 30000 draws: mean 0, variance 1, KS against N(0,1), corner independence.
    Z = np.array([O.normals8(2024, 3, 0, s) for s in range(30000)])
    assert abs(Z.mean()) < 4 / math.sqrt(Z.size)
    assert abs(Z.var() - 1) < 4 * math.sqrt(2 / Z.size)
    assert stats.kstest(Z.ravel(), "norm").pvalue > 1e-3
    C = np.corrcoef(Z.T)
    assert np.abs(C - np.eye(8)).max() < 5 / math.sqrt(30000)


def test_normals_pairwise_independence():
    # R13c draws (z2, z3) from the low 23 bits of word B and the top bytes of A, B, C, while
    # (z0, z1) use the low 23 bits of A and C: a 2-D chi-square over 8 x 8 cells of the
    # probability-integral transform finds no dependence between any two of the eight normals,
    # across samples of all four group positions t
    Z = np.array([O.normals8(99, 12345, 1, s) for s in range(32000)])
    U = stats.norm.cdf(Z)
    for i in range(8):
        for j in range(i + 1, 8):
            H, _, _ = np.histogram2d(U[:, i], U[:, j], bins=8, range=[[0, 1], [0, 1]])
            chi2 = ((H - len(U) / 64) ** 2 / (len(U) / 64)).sum()
            assert stats.chi2.sf(chi2, 63) > 1e-4, (i, j, chi2)
    # and the four positions t of a lane group draw the same distribution
    t = (np.arange(len(Z)) // 32) % 4
    for q in range(4):
        assert stats.kstest(Z[t == q].ravel(), "norm").pvalue > 1e-4, q


# ----------------------------------------------------------------- P5 chol8
def test_chol8_matches_numpy_on_pd():
    g = np.random.default_rng(7)
    for _ in range(20):
        A = g.standard_normal((8, 8))
        S = A @ A.T + 0.1 * np.eye(8)
        assert np.abs(O.chol8(S) - np.linalg.cholesky(S)).max() < 1e-12


def test_chol8_clamps_psd():
    g = np.random.default_rng(8)
    for rank in (1, 3, 5, 7):
        A = g.standard_normal((8, rank))
        S = A @ A.T
        L = O.chol8(S)
        assert np.abs(L @ L.T - S).max() <= 1e-9 * np.diag(S).max()
        assert np.all(np.triu(L, 1) == 0)
        assert np.count_nonzero(np.diag(L)) == rank


# --------------------------------------------------------------------- P9 MC
def test_mc_independent_corners_closed_form():
    # BASELINE pin: diagonal Sigma -> LCP = 1 - prod p_i - prod (1 - p_i).
    g = np.random.default_rng(9)
    N = 40000
    for trial in range(6):
        mu = g.normal(0, 0.7, 8)
        sd = g.uniform(0.3, 1.5, 8)
        th = g.normal(0, 0.3)
        p = stats.norm.cdf((th - mu) / sd)
        want = 1 - np.prod(p) - np.prod(1 - p)
        got = O.mc_count(mu, np.diag(sd), th, N, 77 + trial, trial) / N
        se = math.sqrt(max(want * (1 - want), 1e-12) / N)
        assert abs(got - want) <= 4 * se + 1 / N, (trial, got, want, se)


def test_mc_all_half_closed_form():
    # p_i = 1/2 for all corners: 1 - 2^-7 = 0.9921875
    N = 50000
    got = O.mc_count(np.zeros(8), np.eye(8), 0.0, N, 5, 11) / N
    assert abs(got - 0.9921875) < 4 * math.sqrt(0.9921875 * 0.0078125 / N)


def test_mc_correlated_vs_genz():
    # Library pin: scipy's Genz orthant probabilities for a correlated 8-variate normal.
    g = np.random.default_rng(10)
    N = 40000
    for trial in range(3):
        A = g.standard_normal((8, 8)) * 0.4 + 0.5
        S = A @ A.T / 4 + 0.05 * np.eye(8)
        mu = g.normal(0, 0.5, 8)
        th = 0.1
        mvn = stats.multivariate_normal
        p_below = mvn.cdf(np.full(8, th), mean=mu, cov=S, abseps=1e-6, releps=1e-6,
                          maxpts=2000000, rng=np.random.default_rng(0))
        p_above = mvn.cdf(np.full(8, -th), mean=-mu, cov=S, abseps=1e-6, releps=1e-6,
                          maxpts=2000000, rng=np.random.default_rng(1))
        want = 1 - p_below - p_above
        got = O.mc_count(mu, np.linalg.cholesky(S), th, N, 99, trial) / N
        se = math.sqrt(want * (1 - want) / N)
        assert abs(got - want) <= 4 * se + 2e-4, (got, want, se)


def test_mc_comonotone_is_zero_and_far_cell_zero():
    v = np.linspace(0.5, 1.5, 8)
    S = np.outer(v, v)
    L = O.chol8(S)
    assert O.mc_count(np.full(8, 0.3), L, 0.3, 5000, 1, 2) == 0
    assert O.mc_count(np.full(8, 10.0), np.eye(8), 0.0, 5000, 1, 2) == 0


def test_mc_reflection_and_range_and_determinism():
    g = np.random.default_rng(11)
    A = g.standard_normal((8, 8)) * 0.3
    S = A @ A.T + 0.2 * np.eye(8)
    L = np.linalg.cholesky(S)
    mu = g.normal(0, 0.4, 8)
    N = 40000
    a = O.mc_count(mu, L, 0.2, N, 3, 4) / N
    b = O.mc_count(2 * 1.0 - mu, L, 2 * 1.0 - 0.2, N, 3, 4) / N
    assert abs(a - b) < 5 * math.sqrt(2 * a * (1 - a) / N) + 1e-3
    assert 0 <= a <= 1
    assert O.mc_count(mu, L, 0.2, 1000, 3, 4) == O.mc_count(mu, L, 0.2, 1000, 3, 4)
    assert O.mc_count(mu, L, 0.2, 1000, 3, 4) != O.mc_count(mu, L, 0.2, 1000, 4, 4)


def test_mc_standard_error_scaling():
    # SE of the estimator shrinks ~2x per 4x samples
    mu = np.zeros(8)
    L = np.eye(8) * 0.5
    th = 0.9
    spreads = []
    for N in (400, 6400):
        est = [O.mc_count(mu, L, th, N, seed, 1) / N for seed in range(40)]
        spreads.append(np.std(est))
    ratio = spreads[0] / spreads[1]
    assert 4 / 1.6 < ratio < 4 * 1.6


def _genz_lcp(mu, S, th, seed):
    # LCP = 1 - P(all corners < theta) - P(all corners > theta) (R5),
    # each orthant by scipy's Genz integration of the 8-variate normal
    mvn = stats.multivariate_normal
    kw = dict(cov=S, allow_singular=True, abseps=2e-5, releps=0, maxpts=400000)
    pb = mvn.cdf(np.full(8, th), mean=mu, rng=np.random.default_rng(seed), **kw)
    pa = mvn.cdf(np.full(8, -th), mean=-mu, rng=np.random.default_rng(seed + 1), **kw)
    return 1.0 - pb - pa


@pytest.mark.parametrize("name", ["c1", "t2"])
def test_pmc_cells_composition_vs_genz(name):
    # Pin of the composed leaf estimator orc_pmc_cells (cell posterior -> PI8 corner
    # reorder -> clamped chol8 -> Philox/Box-Muller MC count): on real
    # cell posteriors of the config, with LCP in (0.05, 0.95), the N = 40 000 estimate
    # agrees with Genz orthant probabilities of the same (mu, Sigma) within 4 SE.  A wrong
    # corner permutation, a transposed factor or a dropped Sigma term moves these cells
    # by many SE (the posterior correlations are strong and of both signs).
    from workloads import generate
    w = generate(name)
    cfg = w.cfg
    M = O.Model.from_config(cfg, w.X, w.y)
    th = w.thetas[0]
    ncell = int(np.prod(cfg.cells))
    probe = np.arange(0, ncell, max(1, ncell // 3000), dtype=np.int64)
    coarse = M.pmc_cells(probe, th, 400, 31)
    mid = probe[(coarse > 0.08) & (coarse < 0.92)]
    assert len(mid) >= 12
    cells = np.random.default_rng(5).choice(mid, 12, replace=False)
    N = 40000
    got = M.pmc_cells(cells, th, N, cfg.mc_seed)
    zs = []
    for q, c in enumerate(cells):
        mu, S = M.cell_posterior(int(c))
        want = _genz_lcp(mu, 0.5 * (S + S.T), th, 100 + q)
        assert 0.03 < want < 0.97, (int(c), want)
        se = math.sqrt(want * (1 - want) / N)
        zs.append((got[q] - want) / se)
    zs = np.array(zs)
    assert np.abs(zs).max() <= 4.0, zs
    # the 12 deviations behave like N(0, 1) draws (a biased estimator would shift them)
    assert abs(zs.mean()) <= 4.0 / math.sqrt(len(zs)), zs
