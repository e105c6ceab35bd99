"""Paper-experiment analogues on synthetic fields:
E1/E2: octree-pruned vs pruning-free dense PMC (same local GP, identical Philox
streams): time ratio and RMSE of the LCP fields;
E4: alpha sweep, time vs RMSE (Fig. 5);
E7: level field histogram.
Writes one JSON document to stdout.  Run under gpurun."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_12442_b200 import Context, config_args  # noqa: E402
from workloads import generate  # noqa: E402
from workloads.gen import morton_sorted_cells  # noqa: E402


def timed(fn, reps=3):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = None
    out = None
    for _ in range(reps):
        ev0.record()
        out = fn()
        ev1.record()
        torch.cuda.synchronize()
        t = ev0.elapsed_time(ev1)
        best = t if best is None else min(best, t)
    return best, out


def run(name, alphas):
    w = generate(name)
    cfg = w.cfg
    th = w.thetas[0]
    dev = torch.device("cuda:0")
    kernel, grid, k, b, hf = config_args(cfg)
    ctx = Context(0)
    X = torch.from_numpy(np.array(w.X)).to(dev)
    y = torch.from_numpy(np.array(w.y)).to(dev)
    ctx.fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf)
    ncell = int(np.prod(cfg.cells))
    allc = morton_sorted_cells(cfg.cells, device=dev)   # Morton order: the brick posterior kernels
    lcp_all = torch.empty(ncell, dtype=torch.float32, device=dev)
    field_all = torch.empty(ncell, dtype=torch.float32, device=dev)

    def dense():
        ctx.pmc_cells(allc, th, cfg.n_samples, cfg.mc_seed, 0, out=lcp_all)
        return ctx.scatter_field(allc, lcp_all, field_all)

    t_dense, f_dense = timed(dense)
    f_dense = f_dense.clone()
    level = ctx.set_level_field(torch.empty(ncell, dtype=torch.uint8, device=dev))
    res = {"workload": name, "cells": ncell, "theta": th, "n_samples": cfg.n_samples,
           "dense_local_ms": t_dense, "sweep": []}
    for al in alphas:
        def pruned():
            f, n = ctx.run_field(th, al, cfg.max_depth, cfg.n_samples, cfg.mc_seed, 0)
            return f, n
        t, (f, n) = timed(pruned)
        d = (f.double() - f_dense.double())
        missed = int(((f_dense > al) & (f == 0)).sum())
        hist = torch.bincount(level.long(), minlength=cfg.max_depth + 1)[: cfg.max_depth + 1].tolist()
        res["sweep"].append({"alpha": al, "pruned_ms": t, "time_ratio": t / t_dense, "leaves": n,
                             "leaf_fraction": n / ncell, "rmse": float(d.pow(2).mean().sqrt()),
                             "max_abs_err": float(d.abs().max()), "cells_lcp_gt_alpha_pruned": missed,
                             "level_histogram": hist,
                             "leaves_bitexact_vs_dense": bool(torch.equal(f[f > 0], f_dense[f > 0]))})
    return res


if __name__ == "__main__":
    names = sys.argv[1:] or ["p1", "c3"]
    out = [run(nm, [1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-7]) for nm in names]
    print(json.dumps(out, indent=1))
