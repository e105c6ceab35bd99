"""Exercise every C-ABI entry point on small cases (for compute-sanitizer runs)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_12442_b200 import Context, config_args  # noqa: E402
from workloads import generate  # noqa: E402
from workloads.gen import random_cells  # noqa: E402

dev = torch.device("cuda:0")
for name in ("t1", "t2", "c2"):
    w = generate(name)
    cfg = w.cfg
    kernel, grid, k, b, hf = config_args(cfg)
    ctx = Context(0)
    X = torch.from_numpy(np.array(w.X)).to(dev)
    y = torch.from_numpy(np.array(w.y)).to(dev)
    ctx.fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf, keep_records=True)
    for it, th in enumerate(w.thetas):
        leaves = ctx.octree_refine(th, cfg.alpha, cfg.max_depth)
        rec = ctx.node_records()
        lcp = ctx.pmc_cells(leaves, th, 64, 7, it)
        f = ctx.scatter_field(leaves, lcp)
        f2, n = ctx.run_field(th, cfg.alpha, cfg.max_depth, 64, 7, it)
    cells = torch.from_numpy(random_cells(name, 500, 1)).to(dev)
    mu, cov = ctx.cell_posterior(cells)
    lcp2 = ctx.pmc_cells(cells, w.thetas[0], 33, 9)
    P = torch.rand((100, 3), dtype=torch.float64, device=dev)
    m, v = ctx.point_marginals(P)
    S = ctx.bucket_sets()
    ctx.synchronize()
    print(name, "ok", len(leaves), float(lcp.sum()), float(lcp2.sum()))
# exact GP (k = m) path
w = generate("t1")
kernel, grid, k, b, hf = config_args(w.cfg)
ctx = Context(0).fit_local(torch.from_numpy(np.array(w.X)).to(dev), torch.from_numpy(np.array(w.y)).to(dev),
                           kernel, w.cfg.m, grid, bucket_log2=0)
f, n = ctx.run_field(w.thetas[0], w.cfg.alpha, w.cfg.max_depth, 64, 7)
# NEXT-3 fused multi-isovalue pass (union, masks, k_pmc<T>) and the brick pass opt-out
for name in ("t1", "t2"):
    w = generate(name)
    kernel, grid, k, b, hf = config_args(w.cfg)
    for bp in (0, -1):
        ctx = Context(0).fit_local(torch.from_numpy(np.array(w.X)).to(dev),
                                   torch.from_numpy(np.array(w.y)).to(dev), kernel, k, grid,
                                   bucket_log2=b, h_full=hf, brick_pass=bp)
        th = [w.thetas[0] - 0.2, w.thetas[0], w.thetas[0] + 0.3, 9.0, -9.0]
        fields, nl, nu = ctx.run_field_multi(th, w.cfg.alpha, w.cfg.max_depth, 48, 3, 1)
        cells, mask = ctx.union_cells()
        lcpm = ctx.pmc_cells_multi(cells, th, 40, 5, 2)
        print(name, "multi ok", bp, nu, list(nl), float(fields.sum()), float(lcpm.sum()))
# SGPR input path
w = generate("t2")
kernel, grid, k, b, hf = config_args(w.cfg)
XM = np.array(w.X)[:40]
muM = np.array(w.y)[:40]
AM = np.eye(40) * 1e-3
ctx = Context(0).fit_sgpr(XM, muM, AM, kernel, 16, grid, bucket_log2=b, h_full=hf)
f, n = ctx.run_field(w.thetas[0], w.cfg.alpha, w.cfg.max_depth, 32, 7)
torch.cuda.synchronize()
print("all ok")
