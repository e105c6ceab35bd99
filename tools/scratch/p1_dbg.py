import sys, os; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2512_12442_b200 import Context, config_args
from workloads import generate
w = generate("p1"); cfg = w.cfg; th = w.thetas[0]
dev = torch.device("cuda:0")
kernel, grid, k, b, hf = config_args(cfg)
X = torch.from_numpy(np.array(w.X)).to(dev); y = torch.from_numpy(np.array(w.y)).to(dev)
ctx = Context(0); ctx.fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf)
ncell = int(np.prod(cfg.cells)); allc = torch.arange(ncell, dtype=torch.int64, device=dev)
fd = ctx.pmc_cells(allc, th, cfg.n_samples, cfg.mc_seed, 0).clone()
st = ctx.stats(); print("dense: records", st["pmc_used_records"], "brick_runs", st["brick_runs"])
for al in [1e-1, 1e-3]:
    f, n = ctx.run_field(th, al, cfg.max_depth, cfg.n_samples, cfg.mc_seed, 0)
    st = ctx.stats()
    leaves = ctx.octree_refine(th, al, cfg.max_depth).clone()
    diff = (f[leaves] != fd[leaves])
    print("alpha", al, "leaves", n, "records", st["pmc_used_records"], "fused", st["fused"], "differ", int(diff.sum()), "levels", st["level_nodes"], st["level_refined"])
    if diff.any():
        bad = leaves[diff][:5]
        print("  cells", bad.tolist(), "pruned", f[bad].tolist(), "dense", fd[bad].tolist())
        # recompute these cells through pmc_cells now (records covered?)
        again = ctx.pmc_cells(bad.clone(), th, cfg.n_samples, cfg.mc_seed, 0)
        print("  pmc now", again.tolist(), "records", ctx.stats()["pmc_used_records"])
