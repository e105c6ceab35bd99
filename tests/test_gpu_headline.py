"""Parity on the headline configurations at full size, in the launch configuration
bench.py times (BASELINE north_star tolerances):

* c5 (512^3, the bench workload): node sets and leaf sets of whole level-3 subtrees
  (corner and interior ones) equal the oracle's `subtree=` octree except nodes under
  the 1e-6 band (R19); LCP on >= 1e4 sampled leaves of lcp_run_field within 2/N on
  >= 99.9 % with mean |d| <= 1e-4.
* c4 (256x256x128, three isovalues): per isovalue, the full node set and leaf set
  against the oracle's full octree; >= 1e4 leaf cells per isovalue of the fused
  multi-isovalue field (lcp_run_field_multi, the bench step) at the same LCP bar.
* c3 (128^3): LCP on >= 1e4 leaves of lcp_run_field.

Alg. 1; Eq. 3-4; MC PAPER.md:124-136.
"""
import numpy as np
import pytest

import oracle as O
from parity_util import compare_leaf_sets, compare_node_sets, lcp_parity
from workloads import generate

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

N_LCP = 12000        # sampled leaf cells per comparison (>= 1e4)


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def _fit(name, dev, keep_records):
    from paper_2512_12442_b200 import Context, config_args
    w = generate(name)
    cfg = w.cfg
    kernel, grid, k, b, hf = config_args(cfg)
    ctx = Context(0).fit_local(torch.from_numpy(np.array(w.X)).to(dev), torch.from_numpy(np.array(w.y)).to(dev),
                               kernel, k, grid, bucket_log2=b, h_full=hf, keep_records=keep_records)
    return w, ctx


def _subtree_records(raw, lfull, L0, si, sj, sk):
    """Records (on the device) of the nodes at level >= L0 below node (L0; si, sj, sk)."""
    from paper_2512_12442_b200.lcp import NODE_DTYPE
    I = raw.view(torch.int32).view(-1, NODE_DTYPE.itemsize // 4)
    lv, i, j, k = I[:, 0], I[:, 1], I[:, 2], I[:, 3]
    sh = (lv - L0).clamp(min=0)
    sel = (lv >= L0) & ((i >> sh) == si) & ((j >> sh) == sj) & ((k >> sh) == sk)
    rows = raw.view(-1, NODE_DTYPE.itemsize)[sel]
    return rows.cpu().numpy().reshape(-1).view(NODE_DTYPE)


def _cells_in_box(leaves, cells, lo, side):
    nx, ny = cells[0], cells[1]
    x, y, z = leaves % nx, (leaves // nx) % ny, leaves // (nx * ny)
    m = (x >= lo[0]) & (x < lo[0] + side) & (y >= lo[1]) & (y < lo[1] + side) & (z >= lo[2]) & (z < lo[2] + side)
    return leaves[m]


@pytest.fixture(scope="module")
def c5(dev):
    w, ctx = _fit("c5", dev, keep_records=True)
    M = O.Model.from_config(w.cfg, w.X, w.y)
    return w, ctx, M


def test_c5_subtree_node_and_leaf_sets(c5):
    w, ctx, M = c5
    cfg = w.cfg
    th = w.thetas[0]
    leaves = ctx.octree_refine(th, cfg.alpha, cfg.max_depth)
    raw = ctx.node_records_device()
    lf = M.lfull
    L0 = 3
    side = 1 << (lf - L0)
    report = []
    for s in [(3, 3, 3), (7, 7, 7), (0, 0, 0), (5, 2, 6), (1, 6, 4)]:
        rec_o, leaves_o = M.octree(th, cfg.alpha, cfg.max_depth, subtree=(L0,) + s)
        rec_g = _subtree_records(raw, lf, L0, *s)
        res = compare_node_sets(rec_g, rec_o, cfg.alpha, min_level=L0)
        assert not res["unexcused"], (s, res["unexcused"][:10], res["excused"])
        assert res["max_dU"] < 1e-6, (s, res["max_dU"])
        lo = tuple(side * a for a in s)
        lg = _cells_in_box(leaves, cfg.cells, lo, side).cpu().numpy()
        n_only, n_unex = compare_leaf_sets(lg, leaves_o, res["near"], cfg.cells, lf, cfg.max_depth, min_level=L0)
        assert n_unex == 0, (s, n_only, n_unex)
        if res["excused"] == 0:
            assert np.array_equal(np.sort(lg), leaves_o)
        report.append((s, res["gpu_nodes"], res["oracle_nodes"], res["excused"], len(lg), len(leaves_o), n_only))
    print("c5 subtrees (sub, gpu nodes, oracle nodes, excused, gpu leaves, oracle leaves, differing leaves):",
          report)


def test_c5_lcp_sampled_leaves(c5, dev):
    w, ctx, M = c5
    cfg = w.cfg
    th = w.thetas[0]
    field, n = ctx.run_field(th, cfg.alpha, cfg.max_depth, cfg.n_samples, cfg.mc_seed)
    leaves = ctx.octree_refine(th, cfg.alpha, cfg.max_depth)
    assert len(leaves) == n
    sel = torch.from_numpy(np.sort(np.random.default_rng(11).choice(n, N_LCP, replace=False))).to(dev)
    cells = leaves[sel]
    got = field[cells].cpu().numpy()
    want = M.pmc_cells(cells.cpu().numpy(), th, cfg.n_samples, cfg.mc_seed)
    frac, mean, mx = lcp_parity(got, want, cfg.n_samples)
    print(f"c5 LCP on {N_LCP} leaves: within 2/N {frac:.5f}, mean |d| {mean:.2e}, max {mx:.2e}")
    assert frac >= 0.999 and mean <= 1e-4, (frac, mean, mx)


def test_c4_node_and_leaf_sets_per_isovalue(dev):
    w, ctx = _fit("c4", dev, keep_records=True)
    cfg = w.cfg
    M = O.Model.from_config(cfg, w.X, w.y)
    for th in w.thetas:
        leaves_g = ctx.octree_refine(th, cfg.alpha, cfg.max_depth).cpu().numpy()
        rec_g = ctx.node_records()
        rec_o, leaves_o = M.octree(th, cfg.alpha, cfg.max_depth)
        res = compare_node_sets(rec_g, rec_o, cfg.alpha)
        assert not res["unexcused"], (th, res["unexcused"][:10], res["excused"])
        assert res["max_dU"] < 1e-6, (th, res["max_dU"])
        n_only, n_unex = compare_leaf_sets(leaves_g, leaves_o, res["near"], cfg.cells, M.lfull, cfg.max_depth)
        assert n_unex == 0, (th, n_only, n_unex)
        if res["excused"] == 0:
            assert np.array_equal(np.sort(leaves_g), leaves_o)
        print(f"c4 theta {th}: {res['gpu_nodes']} nodes, {len(leaves_g)} leaves, excused {res['excused']}, "
              f"differing leaves {n_only}")


def test_c4_fused_multi_iso_lcp(dev):
    w, ctx = _fit("c4", dev, keep_records=False)
    cfg = w.cfg
    M = O.Model.from_config(cfg, w.X, w.y)
    thetas = list(w.thetas)
    fields, nl, nu = ctx.run_field_multi(thetas, cfg.alpha, cfg.max_depth, cfg.n_samples, cfg.mc_seed, 0)
    cells_g, mask_g = ctx.union_cells()
    cells_g, mask_g = cells_g.cpu().numpy(), mask_g.cpu().numpy()
    sel = np.sort(np.random.default_rng(3).choice(nu, 13000, replace=False))
    c, mk = cells_g[sel], mask_g[sel]
    want = M.pmc_cells_multi(c, thetas, cfg.n_samples, cfg.mc_seed, 0, mask=mk.astype(np.uint32))
    F = fields.cpu().numpy()
    for t in range(len(thetas)):
        on = ((mk >> t) & 1) == 1
        assert on.sum() >= 10000, (t, int(on.sum()))
        frac, mean, mx = lcp_parity(F[t][c[on]], want[t][on], cfg.n_samples)
        print(f"c4 theta {thetas[t]}: {int(on.sum())} leaf cells, within 2/N {frac:.5f}, mean |d| {mean:.2e}")
        assert frac >= 0.999 and mean <= 1e-4, (t, frac, mean, mx)
        assert np.all(F[t][c[~on]] == 0)


def test_c3_lcp_sampled_leaves(dev):
    w, ctx = _fit("c3", dev, keep_records=False)
    cfg = w.cfg
    M = O.Model.from_config(cfg, w.X, w.y)
    th = w.thetas[0]
    field, n = ctx.run_field(th, cfg.alpha, cfg.max_depth, cfg.n_samples, cfg.mc_seed)
    leaves = ctx.octree_refine(th, cfg.alpha, cfg.max_depth).cpu().numpy()
    _, leaves_o = M.octree(th, cfg.alpha, cfg.max_depth)
    assert np.array_equal(np.sort(leaves), leaves_o)
    cells = np.sort(np.random.default_rng(5).choice(leaves, N_LCP, replace=False))
    got = field.cpu().numpy()[cells]
    want = M.pmc_cells(cells, th, cfg.n_samples, cfg.mc_seed)
    frac, mean, mx = lcp_parity(got, want, cfg.n_samples)
    print(f"c3 LCP on {N_LCP} leaves: within 2/N {frac:.5f}, mean |d| {mean:.2e}, max {mx:.2e}")
    assert frac >= 0.999 and mean <= 1e-4, (frac, mean, mx)
