"""Distribution of the per-cell LCP over the leaves of a workload (GPU): how many cells a
warp-uniform fast path of k_pmc (every sample of a step decided on the cell's majority side)
could take.   python tools/lcp_hist.py c5"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2512_12442_b200 import Context, config_args  # noqa: E402
from workloads import generate  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = generate(name)
cfg = w.cfg
kernel, grid, k, b, hf = config_args(cfg)
dev = torch.device("cuda:0")
ctx = Context(0).fit_local(torch.from_numpy(np.array(w.X)).to(dev), torch.from_numpy(np.array(w.y)).to(dev),
                           kernel, k, grid, bucket_log2=b, h_full=hf)
th = w.thetas[0]
leaves = ctx.octree_refine(th, cfg.alpha, cfg.max_depth)
lcp = ctx.pmc_cells(leaves, th, cfg.n_samples, cfg.mc_seed).double()
edges = [0.0, 1e-12, 1.0 / cfg.n_samples, 1e-3, 1e-2, 0.05, 0.1, 0.5, 0.9, 1.0 - 1e-12, 1.0 + 1e-9]
h = torch.histc(lcp, bins=1, min=0, max=1)  # warm-up of histc
counts = [int(((lcp >= a) & (lcp < b_)).sum()) for a, b_ in zip(edges[:-1], edges[1:])]
st = ctx.stats()
print(json.dumps({"workload": name, "leaves": int(len(leaves)), "mean_lcp": float(lcp.mean()),
                  "edges": edges, "counts": counts, "phase2_frac": st["pmc_phase2_samples"] / (len(leaves) * cfg.n_samples)}))
