import sys, json, numpy as np, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2512_12442_b200 import Context, config_args
from workloads import generate
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
w = generate(name); cfg = w.cfg
kernel, grid, k, b, hf = config_args(cfg)
dev = torch.device("cuda:0")
X = torch.from_numpy(np.array(w.X)).to(dev); y = torch.from_numpy(np.array(w.y)).to(dev)
for slab in ({}, dict(slab_rank=3, slab_count=8)):
    ctx = Context(0).fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf, **slab)
    ctx.octree_refine(w.thetas[0], cfg.alpha, cfg.max_depth)
    for d in range(cfg.max_depth + 1):
        best = 1e9
        for _ in range(3):
            ctx.octree_refine(w.thetas[0], cfg.alpha, d)
            st = ctx.stats(); best = min(best, st["refine_ms"])
        print(name, slab, "max_depth", d, "refine_ms %.3f" % best, "launches", st["launches"], flush=True)
