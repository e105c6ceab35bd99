"""Randomised GPU-vs-oracle parity over the whole path.

Each seed draws a fresh configuration: ragged grid dimensions (including
degenerate 1- and 2-cell axes), an off-origin anisotropic box, SE or Matern-5/2
kernel with random per-axis length scales, nugget and prior mean, m and k, bucket
grid depth, candidate-lattice height, maximum depth, threshold alpha, isovalue
and sample count.  The brick pass, the big-k brick, the record path and the
per-cell path are all reachable from these draws.  Checked against the oracle:
the k-NN sets (bit-exact), the octree node records (R19 band), the leaf sets
and the LCP values of every leaf (R20 statistics, identical Philox streams),
and the fused two-isovalue pass.
"""
import math

import numpy as np
import pytest

import oracle as O
from parity_util import compare_node_sets, lcp_parity, posterior_close

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _draw(seed):
    g = np.random.default_rng(10_000 + seed)
    cells = [int(c) for c in g.integers(3, 41, 3)]
    if seed % 5 == 3:
        cells[int(g.integers(0, 3))] = int(g.integers(1, 3))       # degenerate axis
    lo = g.uniform(-2.0, 1.0, 3)
    hi = lo + g.uniform(0.4, 3.0, 3)
    m = int(g.integers(12, 420))
    X = lo + (hi - lo) * g.random((m, 3))
    nb = 3
    cen = lo + (hi - lo) * g.random((nb, 3))
    amp = g.uniform(-1.0, 1.0, nb)
    wid = g.uniform(0.15, 0.5, nb) * float(np.min(hi - lo))
    d2 = ((X[:, None, :] - cen[None]) ** 2).sum(-1)
    y = (amp * np.exp(-d2 / (2 * wid ** 2))).sum(-1) + 0.3 * (X[:, 2] - lo[2]) / (hi[2] - lo[2])
    y = y + 0.01 * g.standard_normal(m)
    kind = int(g.integers(0, 2))
    var = float(g.uniform(0.3, 2.0))
    ls = tuple(float(v) for v in g.uniform(0.08, 0.5, 3) * (hi - lo))
    nug = float(10 ** g.uniform(-6, -2))
    m0 = float(g.uniform(-0.2, 0.2))
    k = int(g.integers(1, min(m, 200) + 1))
    lfull = max(0, math.ceil(math.log2(max(cells))))
    b = int(g.integers(0, min(lfull, 4) + 1))
    h_full = int(g.integers(0, 4))
    max_depth = int(g.integers(max(0, lfull - 2), lfull + 1))
    alpha = float(10 ** g.uniform(-4, -0.32))
    q = g.uniform(0.25, 0.75, 2)
    thetas = [float(np.quantile(y, q[0])), float(np.quantile(y, q[1]))]
    N = int(g.choice([256, 1000, 2048]))
    return dict(cells=tuple(cells), lo=tuple(lo), hi=tuple(hi), X=X, y=y, kind=kind, var=var, ls=ls,
                nug=nug, m0=m0, k=k, b=b, h_full=h_full, max_depth=max_depth, alpha=alpha,
                thetas=thetas, N=N, seed=int(g.integers(0, 2**31)))


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_whole_path(seed):
    from paper_2512_12442_b200 import Context
    d = _draw(seed)
    dev = torch.device("cuda:0")
    kernel = (d["kind"], d["var"], d["ls"], d["nug"], d["m0"])
    grid = (d["lo"], d["hi"], d["cells"])
    ctx = Context(0)
    ctx.fit_local(torch.from_numpy(d["X"]).to(dev), torch.from_numpy(d["y"]).to(dev), kernel, d["k"], grid,
                  bucket_log2=d["b"], h_full=d["h_full"], keep_records=True)
    M = O.Model(O.make_kernel(d["kind"], d["var"], d["ls"], d["nug"], d["m0"]),
                O.make_grid(d["lo"], d["hi"], d["cells"]), d["X"], d["y"], d["k"], d["b"], d["h_full"])
    S = ctx.bucket_sets().cpu().numpy()
    for bk in range(M.nbuckets):
        np.testing.assert_array_equal(S[bk], M.bucket_set(bk))
    th, alpha, md, N = d["thetas"][0], d["alpha"], d["max_depth"], d["N"]
    leaves = ctx.octree_refine(th, alpha, md).clone()
    rec_o, leaves_o = M.octree(th, alpha, md)
    res = compare_node_sets(ctx.node_records(), rec_o, alpha)
    assert not res["unexcused"], (d, res["unexcused"][:10])
    assert res["max_dU"] < 1e-6, res
    lv = leaves.cpu().numpy()
    if res["excused"] == 0:
        np.testing.assert_array_equal(np.sort(lv), leaves_o)
    if len(lv):
        sel = np.random.default_rng(seed).choice(len(lv), min(64, len(lv)), replace=False)
        mu_g, cov_g = ctx.cell_posterior(leaves[torch.from_numpy(sel).to(dev)])
        mu_g, cov_g = mu_g.cpu().numpy(), cov_g.cpu().numpy()
        for q, c in enumerate(lv[sel]):
            mu_o, cov_o = M.cell_posterior(int(c))
            em, ec = posterior_close(mu_g[q], mu_o, cov_g[q], cov_o, d["var"], 1e-5)
            assert em <= 1e-5 and ec <= 1e-5, (int(c), em, ec)
    lcp_g = ctx.pmc_cells(leaves, th, N, d["seed"]).cpu().numpy()
    lcp_o = M.pmc_cells(lv, th, N, d["seed"])
    frac, mean, mx = lcp_parity(lcp_g, lcp_o, N)
    assert frac >= 0.999 and mean <= 1e-4, (frac, mean, mx)
    f, nl = ctx.run_field(th, alpha, md, N, d["seed"])
    assert nl == len(lv)
    assert torch.equal(f[leaves], torch.from_numpy(lcp_g).to(dev))
    # fused two-isovalue pass over the union of the two leaf sets
    fields, nls, nu = ctx.run_field_multi(d["thetas"], alpha, md, N, d["seed"], 2)
    cells_u, mask_u = ctx.union_cells()
    cells_u, mask_u = cells_u.cpu().numpy(), mask_u.cpu().numpy()
    assert len(cells_u) == nu
    if len(cells_u):
        lcp_m = M.pmc_cells_multi(cells_u, d["thetas"], N, d["seed"], 2, mask=mask_u.astype(np.uint32))
        F = fields.cpu().numpy()
        for t in range(2):
            frac, mean, mx = lcp_parity(F[t][cells_u], lcp_m[t], N)
            assert frac >= 0.999 and mean <= 1e-4, (t, frac, mean, mx)


def _opts(seed, d):
    """Option draws for the second sweep: local-set mode, extreme search, FP32
    posterior, brick-pass opt-out, number of isovalues."""
    g = np.random.default_rng(20_000 + seed)
    o = dict(local_mode=int(g.random() < 0.35), beta=float(g.uniform(0.3, 2.0)),
             extreme_iters=int(g.choice([0, 0, 16, 48])), brick_pass=-1 if g.random() < 0.3 else 0,
             precision=int(g.random() < 0.25))
    if o["local_mode"]:
        m = len(d["y"])
        o["k"] = m if g.random() < 0.6 else int(g.integers(max(1, d["k"] // 2), m + 1))
    else:
        o["k"] = d["k"]
    if o["k"] > 128:
        o["precision"] = 0   # the FP32 posterior needs k <= 128 (EINVAL otherwise)
    T = int(g.integers(1, 6))
    o["thetas"] = [float(v) for v in np.quantile(d["y"], np.sort(g.uniform(0.2, 0.8, T)))]
    if o["precision"]:
        d = dict(d, nug=max(d["nug"], 1e-3))
    return o, d


@pytest.mark.parametrize("seed", range(30))
def test_fuzz_options(seed):
    from paper_2512_12442_b200 import Context, LcpError
    d0 = _draw(100 + seed)
    o, d = _opts(seed, d0)
    dev = torch.device("cuda:0")
    kernel = (d["kind"], d["var"], d["ls"], d["nug"], d["m0"])
    grid = (d["lo"], d["hi"], d["cells"])
    kern_o = O.make_kernel(d["kind"], d["var"], d["ls"], d["nug"], d["m0"])
    grid_o = O.make_grid(d["lo"], d["hi"], d["cells"])
    k = o["k"]
    err_o = err_g = None
    try:
        if o["local_mode"]:
            M = O.Model.box(kern_o, grid_o, d["X"], d["y"], k, d["b"], d["h_full"], o["beta"])
        else:
            M = O.Model(kern_o, grid_o, d["X"], d["y"], k, d["b"], d["h_full"])
    except O.OracleError as e:
        err_o = e.status
    ctx = Context(0)
    try:
        ctx.fit_local(torch.from_numpy(d["X"]).to(dev), torch.from_numpy(d["y"]).to(dev), kernel, k, grid,
                      bucket_log2=d["b"], h_full=d["h_full"], keep_records=True,
                      extreme_iters=o["extreme_iters"], brick_pass=o["brick_pass"],
                      local_mode=o["local_mode"], beta=o["beta"], precision=o["precision"])
    except LcpError as e:
        err_g = e.status
    assert err_o == err_g, (o, err_o, err_g)
    if err_o is not None:
        return
    M.set_extreme(o["extreme_iters"])
    S = ctx.bucket_sets().cpu().numpy()
    for bk in range(M.nbuckets):
        np.testing.assert_array_equal(S[bk], M.bucket_set(bk))
    tol = 1e-4 if o["precision"] else 1e-5
    frac_min = 0.995 if o["precision"] else 0.999
    alpha, md, N = d["alpha"], d["max_depth"], d["N"]
    thetas = o["thetas"]
    for th in thetas[:2]:
        leaves = ctx.octree_refine(th, alpha, md).clone()
        rec_o, leaves_o = M.octree(th, alpha, md)
        res = compare_node_sets(ctx.node_records(), rec_o, alpha)
        assert not res["unexcused"], (o, res["unexcused"][:10])
        assert res["max_dU"] < 1e-6, res
        lv = leaves.cpu().numpy()
        if res["excused"] == 0:
            np.testing.assert_array_equal(np.sort(lv), leaves_o)
        if len(lv):
            sel = np.random.default_rng(seed).choice(len(lv), min(48, len(lv)), replace=False)
            mu_g, cov_g = ctx.cell_posterior(leaves[torch.from_numpy(sel).to(dev)])
            mu_g, cov_g = mu_g.cpu().numpy(), cov_g.cpu().numpy()
            for q, c in enumerate(lv[sel]):
                mu_o, cov_o = M.cell_posterior(int(c))
                em, ec = posterior_close(mu_g[q], mu_o, cov_g[q], cov_o, d["var"], tol)
                assert em <= tol and ec <= tol, (o, int(c), em, ec)
    fields, nls, nu = ctx.run_field_multi(thetas, alpha, md, N, d["seed"], 5)
    cells_u, mask_u = ctx.union_cells()
    cells_u, mask_u = cells_u.cpu().numpy(), mask_u.cpu().numpy()
    assert len(cells_u) == nu
    F = fields.cpu().numpy()
    if len(cells_u):
        lcp_m = M.pmc_cells_multi(cells_u, thetas, N, d["seed"], 5, mask=mask_u.astype(np.uint32))
        for t in range(len(thetas)):
            frac, mean, mx = lcp_parity(F[t][cells_u], lcp_m[t], N)
            assert frac >= frac_min and mean <= 1e-4, (o, t, frac, mean, mx)
    for t in range(len(thetas)):
        off = np.ones(F.shape[1], bool)
        off[cells_u[(mask_u >> t) & 1 == 1]] = False
        assert np.all(F[t][off] == 0)
