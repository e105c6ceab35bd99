#!/usr/bin/env python
"""Per-rank work of the z-slab decomposition, measured on ONE GPU by
running each rank's step alone, one after another: every rank's context fits with
slab_rank / slab_count (automatic level, weighted cuts) and runs the bench step
(fit + lcp_run_field, or the fused lcp_run_field_multi).  Reports per-rank leaf
cells and device step times, the leaf max/mean imbalance, and the efficiency the
partition allows, T_1 / (N max_r T_r) -- a projection from per-rank times, not a
multi-GPU measurement (no concurrent ranks, no interconnect).

    python tools/slab_balance.py c4 c5 p1 --ranks 2 4 8 --out profiles/r2_slab_balance.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="+")
    ap.add_argument("--ranks", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--out", default=None)
    ap.add_argument("--fit-shard", action="store_true",
                    help="the bucket factors split across the ranks (dist.fit_sharded); the all-gather is "
                         "emulated by copies between the ranks' contexts and its NVLink time modelled")
    args = ap.parse_args()
    import torch

    from paper_2512_12442_b200 import Context, config_args
    from workloads import generate
    dev = torch.device("cuda:0")
    res = {}
    for name in args.workloads:
        w = generate(name)
        cfg = w.cfg
        kernel, grid, k, b, hf = config_args(cfg)
        X = torch.from_numpy(np.array(w.X)).to(dev)
        y = torch.from_numpy(np.array(w.y)).to(dev)
        T = len(w.thetas)

        def step(ctx, slab):
            ctx.fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf, **slab)
            if T > 1:
                _, nl, _ = ctx.run_field_multi(list(w.thetas), cfg.alpha, cfg.max_depth, cfg.n_samples, cfg.mc_seed, 0)
                return int(np.sum(nl))
            return ctx.run_field(w.thetas[0], cfg.alpha, cfg.max_depth, cfg.n_samples, cfg.mc_seed)[1]

        def timed(ctx, slab):
            best = None
            for _ in range(args.reps):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                n = step(ctx, slab)
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1)
                best = t if best is None else min(best, t)
            return n, best, ctx.stats()

        def sharded(N):
            """Every rank's sharded fit (timed), the in-place all-gather emulated by device copies
            between the ranks' contexts (not timed; modelled as 7/8 of the blocks over NVLink at
            700 GB/s), then each rank's lcp_fit_finish + run_field (timed)."""
            ctxs = [Context(0) for _ in range(N)]
            for rnd in range(2):               # round 0 warms the contexts (allocations), round 1 is timed
                t_fit = []
                for r in range(N):
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    ctxs[r].fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf, slab_rank=r, slab_count=N,
                                      fit_shard=1)
                    e1.record()
                    torch.cuda.synchronize()
                    t_fit.append(e0.elapsed_time(e1))
                bufs = [c_.fit_shard_buffers() for c_ in ctxs]
                for r in range(N):             # the all-gather
                    for dst in range(N):
                        if dst != r:
                            for which in (0, 2):
                                ch = bufs[r][which + 1]
                                bufs[dst][which][r * ch:(r + 1) * ch].copy_(bufs[r][which][r * ch:(r + 1) * ch])
                torch.cuda.synchronize()
                gather_bytes = (N - 1) * (bufs[0][1] + bufs[0][3])
                t_gather = gather_bytes / 700e9 * 1e3
                del bufs
                leaves, times = [], []
                for r in range(N):
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    ctxs[r].fit_finish()
                    if T > 1:
                        _, nl, _ = ctxs[r].run_field_multi(list(w.thetas), cfg.alpha, cfg.max_depth, cfg.n_samples,
                                                           cfg.mc_seed, 0)
                        n = int(np.sum(nl))
                    else:
                        n = ctxs[r].run_field(w.thetas[0], cfg.alpha, cfg.max_depth, cfg.n_samples, cfg.mc_seed)[1]
                    e1.record()
                    torch.cuda.synchronize()
                    leaves.append(n)
                    times.append(t_fit[r] + e0.elapsed_time(e1) + t_gather)
            del ctxs
            torch.cuda.empty_cache()
            assert sum(leaves) == n1, (name, N, leaves, n1)
            L = np.array(leaves, float)
            tm = np.array(times)
            print(f"{name} N={N} sharded fit: fit ms {[round(x, 2) for x in t_fit]}, modelled all-gather "
                  f"{t_gather:.2f} ms ({gather_bytes / 1e9:.2f} GB per rank); step ms {[round(x, 1) for x in times]} "
                  f"(T1 {t1:.1f}) -> projected efficiency {t1 / (N * tm.max()):.3f}", flush=True)
            return {"fit_shard": True, "fit_ms_per_rank": [round(x, 3) for x in t_fit],
                    "modelled_allgather_ms": t_gather, "allgather_bytes_per_rank": gather_bytes,
                    "leaves_per_rank": leaves, "leaf_max_over_mean": float(L.max() / L.mean()),
                    "step_ms_per_rank": [round(x, 3) for x in times],
                    "projected_efficiency": float(t1 / (N * tm.max()))}

        phase_keys = ("fit_ms", "refine_ms", "brick_pass_ms", "posterior_ms", "chol_ms", "mc_ms", "scatter_ms",
                      "launches", "vertex_marginals")

        def phases(st):
            return {key: st[key] for key in phase_keys if key in st}

        one = Context(0)
        step(one, {})
        n1, t1, st1 = timed(one, {})
        one_leaves = [one.octree_refine(th, cfg.alpha, cfg.max_depth).cpu().numpy() for th in w.thetas[:1]]
        lf = one.info()["lfull"]
        del one
        out = {"leaves_n1": n1, "t1_ms": t1, "phases_n1": phases(st1), "ranks": {}}
        for N in args.ranks:
            if args.fit_shard:
                out["ranks"][N] = sharded(N)
                continue
            leaves, times, plan, ph = [], [], None, []
            for r in range(N):
                ctx = Context(0)
                step(ctx, dict(slab_rank=r, slab_count=N))   # warm-up
                n, t, st = timed(ctx, dict(slab_rank=r, slab_count=N))
                leaves.append(n)
                times.append(t)
                plan = st["slab"]
                ph.append(phases(st))
                del ctx
                torch.cuda.empty_cache()
            assert sum(leaves) == n1, (name, N, leaves, n1)
            L = np.array(leaves, float)
            tm = np.array(times)
            # leaf cells of the first isovalue per z-layer of the slab level (N = 1 run), beside the weights
            lv = one_leaves[0]
            side = 1 << (lf - plan["level"])
            per_layer = np.bincount(lv // (cfg.cells[0] * cfg.cells[1]) // side, minlength=plan["layers"])
            out["ranks"][N] = {"slab_level": plan["level"], "layers": plan["layers"], "layer_cuts": plan["layer_cuts"],
                               "weights": plan["weights"], "leaves_theta0_per_layer": per_layer.tolist(),
                               "leaves_per_rank": leaves, "leaf_max_over_mean": float(L.max() / L.mean()),
                               "step_ms_per_rank": [round(x, 3) for x in times],
                               "projected_efficiency": float(t1 / (N * tm.max())),
                               "empty_ranks": int((L == 0).sum()), "phases_per_rank": ph}
            print(f"{name} N={N}: level {plan['level']} ({plan['layers']} layers) cuts {plan['layer_cuts']} "
                  f"leaves {leaves} max/mean {L.max() / L.mean():.3f}; step ms {[round(x, 1) for x in times]} "
                  f"(T1 {t1:.1f}) -> projected efficiency {t1 / (N * tm.max()):.3f}", flush=True)
        res[name] = out
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
