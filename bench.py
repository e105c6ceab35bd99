#!/usr/bin/env python
"""Benchmark of the LCP hot path (BASELINE.json metric: PMC LCP cells/sec and
end-to-end octree LCP time at 1/2/4/8 B200; % FP32 roofline).

One step = one pass of the whole hot path over the
workload: lcp_fit_local (binning, k-NN, bucket factors, observation marginals)
+ lcp_run_field (octree refine, leaf posterior, chol8, Philox MC, dense field
scatter) and, for N > 1 GPUs, the NCCL reduction of the per-slab fields to rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5] [--impl ours|reference]

Rank 0 prints ONE JSON line.  See DESIGN.md §6 for every key.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PMC LCP cells/sec"
UNIT = "cells/s"
# minimal op mix of the two-phase k_pmc, in issue slots (lane-ops):
#   phase 1, every sample : 3/4 of a Philox4x32-10 block 30 (R13c: 3 blocks per 4 samples),
#                           top-byte gather 2 PRMT, 2 Box-Muller pairs 20 (8 MUFU),
#                           partial L z 26 FFMA, bounds 8, min/max 12, decision 5, queue 3  = 106
#                           (cuobjdump -sass of k_pmc<1>: 429 instructions per 128-sample group)
#   phase 2, queued sample: Philox 40, 2 Box-Muller pairs 20, 10 FFMA, min/max 6,
#                           decision 3, queue store + load 14                              =  93
OPS_PHASE1 = 106
OPS_PHASE2 = 93
# each further isovalue of a fused pass (k_pmc<T>, cuobjdump -sass: 271 vs 210 instructions per
# two-sample phase-1 iteration at T = 3 vs 1): + 15 per sample; its crossing test in phase 2: + 4
OPS_PHASE1_PER_EXTRA_ISO = 15
OPS_PHASE2_PER_EXTRA_ISO = 4
# SURVEY.md §8(d) per-unit figure of the leaf MC ("minimal op mix", fixed before any kernel):
# 170-210 CUDA-core issue slots + 16 MUFU per sample; the lower end, 186, is used, and each
# further isovalue of a fused multi-isovalue pass adds the crossing-test row (21 slots).
OPS_SURVEY = 186
OPS_SURVEY_PER_EXTRA_ISO = 21
SM_COUNT = 148
try:
    HBM_PEAK_GBS = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    HBM_PEAK_GBS = 6532.9
LANES_PER_SM_CLK = 128


# BASELINE.json asks for the paper's quoted timings beside ours, as context only (hardware unstated
# in the paper; C++/Cython/Python on a CPU; N = 1600 samples)
PAPER_CONTEXT = {
    "hardware": "unstated in the paper (CPU implementation, PAPER.md:303)",
    "dense_reconstruction_m500_128cube": "> 16 min (PAPER.md:15)",
    "table3_dense_pmc_m500": "1232 s; ours (pruned) 249 s (PAPER.md:459-462)",
    "table2_ours_by_resolution": "64: 46.7 s, 128: 4.2 min, 256: 20.3 min, 512: 2.17 h, 1024: 14.1 h (PAPER.md:440-442)",
    "table2_dense_by_resolution": "64: 156.5 s, 128: 20.9 min, 256: 164.9 min, 512: 22.0 h (extrapolated) (PAPER.md:443)",
    "cited_pmc_256x256x128": "~45 min (original PMC paper, cited at PAPER.md:17)",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-fit-shard", action="store_true",
                    help="N > 1: every rank fits every bucket (default: factors sharded and all-gathered)")
    ap.add_argument("--extreme", type=int, default=0,
                    help="NEXT-1: continuous extreme-search iterations at coarse octree nodes (0 = lattice)")
    ap.add_argument("--separate-iso", action="store_true",
                    help="multi-isovalue workloads: one run_field per isovalue instead of the fused NEXT-3 pass")
    ap.add_argument("--dense", choices=["exact", "local"], default=None,
                    help="pruning-free baseline, PMC of every cell: 'exact' = exact GP (k = m, one bucket; "
                         "BASELINE c3), 'local' = the configured bucket-local GP (isolates the pruning)")
    return ap.parse_args()


def workload_desc(cfg, thetas):
    kern = {0: "SE", 1: "Matern-5/2"}[cfg.kernel]
    return (f"{cfg.name}: {cfg.cells[0]}x{cfg.cells[1]}x{cfg.cells[2]} cells, m={cfg.m} observations "
            f"({cfg.placement}), {cfg.n_bumps} Gaussian bumps, {kern} l={cfg.lengthscale[0]} "
            f"var={cfg.variance} nugget={cfg.nugget}, k={cfg.k}, bucket_log2={cfg.bucket_log2}, "
            f"h_full={cfg.h_full}, N={cfg.n_samples}, alpha={cfg.alpha}, max_depth={cfg.max_depth}, "
            f"isovalues={thetas}")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_traffic(cells_per_launch, kernel="k_pmc"):
    """DRAM bytes per launch of the dominant kernel: the per-cell traffic of an
    `ncu --set full` capture (profiles/traffic.json) times the cells one bench launch
    processes (k_pmc is one launch over all leaves)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(p))[kernel]["dram_bytes_per_cell"] * cells_per_launch
    except Exception:
        return None


def sample_subtrees(cfg, lfull):
    """BASELINE.md §3 sample of the oracle arm: the level-3 octree subtrees with z-index 0
    (1/8 of the domain), visited in a fixed co-prime order so that consecutive steps
    land in different places (corner, edge and interior subtrees).  Grids of at most
    2^21 cells (c1-c3) are sampled whole (subtree None)."""
    if int(np.prod(cfg.cells)) <= (1 << 21) or cfg.max_depth < 3:
        return [None]
    side = 1 << (lfull - 3)
    ni, nj = [-(-cfg.cells[d] // side) for d in (0, 1)]
    subs = [(3, i, j, 0) for j in range(nj) for i in range(ni)]
    n = len(subs)
    stride = next(s for s in (37, 29, 23, 19, 17, 13, 11, 7, 5, 3, 1) if np.gcd(s, n) == 1)
    return [subs[(q * stride) % n] for q in range(n)]


ORACLE_LEAVES_PER_STEP = 4000


def oracle_step(w, M, sub):
    """One step of the oracle arm on a bounded sample, timed as it runs: the oracle's octree
    (Alg. 1) on subtree `sub` (None = the whole grid) for every isovalue, then its leaf pass
    (posterior, chol8, MC) on at most ORACLE_LEAVES_PER_STEP evenly spaced leaves of it.
    Returns (measured seconds, leaf cells of the sample over all isovalues, seconds of
    the octree, seconds and cells of the leaf pass)."""
    cfg = w.cfg
    t_oct = t_pmc = 0.0
    n_leaf = n_pmc = 0
    t_start = time.perf_counter()
    for it, th in enumerate(w.thetas):
        t0 = time.perf_counter()
        _, leaves = M.octree(th, cfg.alpha, cfg.max_depth, subtree=sub)
        t_oct += time.perf_counter() - t0
        pick = leaves[np.unique(np.linspace(0, len(leaves) - 1, min(len(leaves), ORACLE_LEAVES_PER_STEP)).astype(
            np.int64))] if len(leaves) else leaves
        t0 = time.perf_counter()
        if len(pick):
            M.pmc_cells(pick, th, cfg.n_samples, cfg.mc_seed, it)
        t_pmc += time.perf_counter() - t0
        n_leaf += len(leaves)
        n_pmc += len(pick)
    return time.perf_counter() - t_start, n_leaf, t_oct, t_pmc, n_pmc


def oracle_rate(cfg, M, t_fit, secs_oct, secs_pmc, n_leaf, n_pmc, sub_cells):
    """Leaf cells/s of the oracle's whole path estimated from measured parts: seconds per
    leaf cell of the octree (sample subtree) + of the leaf pass (its sampled leaves) + the
    model build amortised by the sample's share of the grid."""
    total = int(np.prod(cfg.cells))
    per_leaf = (secs_oct / max(n_leaf, 1) + secs_pmc / max(n_pmc, 1)
                + t_fit * (sub_cells / total) / max(n_leaf, 1))
    return 1.0 / per_leaf


def _sub_cells(cfg, lfull, sub):
    if sub is None:
        return int(np.prod(cfg.cells))
    side = 1 << (lfull - sub[0])
    return int(np.prod([max(0, min(side, cfg.cells[d] - side * sub[1 + d])) for d in range(3)]))


def hbm_fractions(cells_per_launch, s_per_launch):
    """HBM bandwidth of the hot kernels vs the measured copy peak (MEASURED_PEAKS.json):
    k_pmc from its ncu bytes per cell x this run's cells / this run's k_pmc time; the
    brick-pass kernels from their own ncu capture (profiles/traffic.json)."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except Exception:
        return None
    peak = HBM_PEAK_GBS
    out = {"peak_gbs": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"}
    if s_per_launch > 0:
        gbs = t["k_pmc"]["dram_bytes_per_cell"] * cells_per_launch / s_per_launch / 1e9
        out["k_pmc"] = {"gbs": gbs, "frac": gbs / peak, "source": "ncu bytes/cell x live time"}
    for kname in ("k_brick", "k_chol8_rec"):
        if kname in t:
            out[kname] = {"gbs": t[kname]["ncu_gbs"], "frac": t[kname]["ncu_hbm_frac"], "source": "ncu capture"}
    return out


def oracle_sample(w, steps=1, warmup=0):
    """Oracle arm: build the model once (timed), then `warmup + steps` sample steps.
    Returns (value, measured seconds per timed step, detail dict)."""
    import oracle as O
    cfg = w.cfg
    t0 = time.perf_counter()
    M = O.Model.from_config(cfg, w.X, w.y)
    t_fit = time.perf_counter() - t0
    subs = sample_subtrees(cfg, M.lfull)
    secs = []
    acc = [0.0, 0.0, 0, 0, 0]
    visited = []
    for s in range(warmup + steps):
        sub = subs[s % len(subs)]
        dt, n_leaf, t_oct, t_pmc, n_pmc = oracle_step(w, M, sub)
        if s >= warmup:
            secs.append(dt)
            for q, v in enumerate((t_oct, t_pmc, n_leaf, n_pmc, _sub_cells(cfg, M.lfull, sub))):
                acc[q] += v
            visited.append(sub)
    value = oracle_rate(cfg, M, t_fit, acc[0], acc[1], acc[2], acc[3], acc[4])
    total_leaf_est = acc[2] * int(np.prod(cfg.cells)) / max(acc[4], 1)
    where = ("the whole grid" if subs[0] is None else
             f"level-3 subtrees (L, i, j, k) {visited[:6]}{' ...' if len(visited) > 6 else ''} of the z-index-0 "
             f"layer (BASELINE.md §3; {len(subs)} subtrees = 1/8 of the domain)")
    detail = {"sample": (f"oracle (C, FP64, OpenMP) per step: octree (Alg. 1) on {where}, every isovalue; "
                         f"leaf pass on <= {ORACLE_LEAVES_PER_STEP} evenly spaced leaves of it; model build "
                         f"{t_fit:.2f} s once, amortised by the sample's share of the grid"),
              "measured_s_per_step": float(np.mean(secs)) if secs else None,
              "octree_s": acc[0], "leaf_pass_s": acc[1], "leaf_cells_in_sample": acc[2],
              "leaf_pass_cells": acc[3], "sample_grid_cells": acc[4], "model_build_s": t_fit,
              "extrapolated_full_workload_s": total_leaf_est / value if value else None}
    return value, (float(np.mean(secs)) if secs else 0.0), detail


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as O
    from workloads import generate
    w = generate(args.workload)
    cfg = w.cfg
    cores = O.num_threads()
    value, s_step, detail = oracle_sample(w, args.steps, args.warmup)
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * s_step,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": workload_desc(cfg, w.thetas), "sample": detail["sample"]},
           "value_note": ("leaf cells/s of the oracle's whole path, from the measured per-leaf seconds of "
                          "its octree and leaf pass on the sample; ms_per_step is the measured time of one "
                          "sample step"),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                            "sample": detail["sample"]},
           "oracle_detail": detail,
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2512_12442_b200 import Context, config_args
    from paper_2512_12442_b200.dist import cell_ranges, equal_z_cuts, fit_sharded, gather_fields, plan_z_cuts
    from workloads import generate

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_DIST_BACKEND=gloo (functional check of the N > 1 path on fewer GPUs than ranks:
    # ranks share devices round-robin, collectives go through host copies; not a measurement)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count() if backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def all_reduce(x, op):
        if backend == "gloo":
            h = x.cpu()
            dist.all_reduce(h, op=op)
            x.copy_(h)
        else:
            dist.all_reduce(x, op=op)
    w = generate(args.workload)
    cfg = w.cfg
    kernel, grid, k, b, hf = config_args(cfg)
    X = torch.from_numpy(np.array(w.X)).to(dev)
    y = torch.from_numpy(np.array(w.y)).to(dev)
    ncell = int(np.prod(cfg.cells))
    field = torch.empty(ncell, dtype=torch.float32, device=dev)
    multi_fields = (torch.empty((len(w.thetas), ncell), dtype=torch.float32, device=dev)
                    if len(w.thetas) > 1 else None)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    slab = dict(slab_rank=rank, slab_count=world) if world > 1 else {}   # automatic slab level (lcp.h)
    if args.dense:
        # pruning-free baseline (BASELINE c3): exact GP (k = m, one bucket), every cell of the slab
        if args.dense == "exact":
            k, b = cfg.m, 0
        dense_cuts = equal_z_cuts(cfg.cells, world, cfg.max_depth) if world > 1 else [0, cfg.cells[2]]
        c0, c1 = cell_ranges(cfg.cells, dense_cuts)[rank if world > 1 else 0]
        from workloads.gen import morton_sorted_cells
        dense_cells = morton_sorted_cells(cfg.cells, c0, c1, device=dev)   # brick-kernel order
        dense_lcp = torch.empty(c1 - c0, dtype=torch.float32, device=dev)
    ctx = Context(local)
    if world > 1:
        dist.barrier()   # every rank joins the group's first collective

    def barrier():
        if world > 1:
            dist.barrier()

    def step(host=None):
        """fit + run_field for every isovalue; returns (leaf cells summed over the isovalues,
        k_pmc ms, phase-2 samples, leaf cells of the union of isovalues).  host = (X, y, field)
        numpy arrays in pinned memory: the e2e leg, inputs and the output field through the
        C ABI's host-pointer paths (at N > 1 the gathered field is read back on rank 0)."""
        xin, yin = (X, y) if host is None else (host[0], host[1])
        if world > 1 and not args.no_fit_shard:
            # the bucket factors split across the ranks and all-gathered in place (NCCL)
            fit_sharded(ctx, xin, yin, kernel, k, grid, rank, world, bucket_log2=b, h_full=hf,
                        extreme_iters=args.extreme)
        else:
            ctx.fit_local(xin, yin, kernel, k, grid, bucket_log2=b, h_full=hf, extreme_iters=args.extreme, **slab)
        abi_host_out = host is not None and world == 1
        leaves = 0
        mc_ms = 0.0
        p2 = 0
        if len(w.thetas) > 1 and not args.dense and not args.separate_iso:
            # NEXT-3: all isovalues in one fused leaf pass (one posterior, one sample stream)
            fields_out = host[2].reshape(len(w.thetas), ncell) if abi_host_out else multi_fields
            _, nl, nu = ctx.run_field_multi(list(w.thetas), cfg.alpha, cfg.max_depth, cfg.n_samples, cfg.mc_seed,
                                            0, fields=fields_out)
            st = ctx.stats()
            if world > 1:
                gather_fields(fields_out, cfg.cells, plan_z_cuts(st))
            if host is not None and not abi_host_out and rank == 0:
                host[2].reshape(len(w.thetas), ncell)[:] = fields_out.cpu().numpy()
            return int(np.sum(nl)), st["mc_ms"], st["pmc_phase2_samples"], int(nu)
        for it, th in enumerate(w.thetas):
            if args.dense:
                ctx.pmc_cells(dense_cells, th, cfg.n_samples, cfg.mc_seed, it, out=dense_lcp)
                out = ctx.scatter_field(dense_cells, dense_lcp, field)
                if abi_host_out:
                    host[2][:] = out.cpu().numpy()
                n = len(dense_cells)
            else:
                _, n = ctx.run_field(th, cfg.alpha, cfg.max_depth, cfg.n_samples, cfg.mc_seed, it,
                                     field=host[2] if abi_host_out else field)
            leaves += n
            st = ctx.stats()
            mc_ms += st["mc_ms"]
            p2 += st["pmc_phase2_samples"]
            if world > 1:   # slab slices -> rank 0
                gather_fields(field, cfg.cells, dense_cuts if args.dense else plan_z_cuts(st))
                if host is not None and rank == 0:
                    host[2][:] = field.cpu().numpy()
        return leaves, mc_ms, p2, leaves

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = ctx.stats()["launches"]
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    total_ms = 0.0
    leaves_tot = 0
    union_tot = 0
    mc_ms_tot = 0.0
    p2_tot = 0
    st_phase = {"fit_ms": 0.0, "refine_ms": 0.0, "brick_pass_ms": 0.0, "posterior_ms": 0.0, "chol_ms": 0.0,
                "mc_ms": 0.0}
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for _ in range(args.steps):
        flush.fill_(1)                      # L2 flush between timed steps (256 MB > 126 MB L2)
        torch.cuda.synchronize()
        e0.record()
        leaves, mc_ms, p2, union = step()
        e1.record()
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
        leaves_tot += leaves
        union_tot += union
        mc_ms_tot += mc_ms
        p2_tot += p2
        s = ctx.stats()
        for key in st_phase:
            st_phase[key] += s[key] if key != "mc_ms" else 0.0
    st_phase["mc_ms"] = mc_ms_tot
    barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = ctx.stats()["launches"] - launches0
    t = torch.tensor([total_ms, mc_ms_tot], dtype=torch.float64, device=dev)
    lv = torch.tensor([leaves_tot, launches, p2_tot, union_tot], dtype=torch.float64, device=dev)
    if world > 1:
        all_reduce(t, dist.ReduceOp.MAX)
        all_reduce(lv, dist.ReduceOp.SUM)
    total_ms = float(t[0])
    ms_step = total_ms / args.steps
    cells_per_step = ncell * len(w.thetas)
    leaves_step = float(lv[0]) / args.steps          # leaf cells x isovalues: LCP values produced
    union_step = float(lv[3]) / args.steps           # cells through k_pmc (the fused pass tests T isovalues)
    # BASELINE metric "PMC LCP cells/sec": leaf cells (LCP values) of the whole job per second
    # of the end-to-end step (fit + octree + leaf pass + scatter [+ gather])
    value = leaves_step / (ms_step / 1000.0)
    samples_step = union_step * cfg.n_samples

    # e2e: the same step through the C ABI with host (pinned) buffers: X, y in through
    # lcp_fit_local's host path, the LCP field(s) out through lcp_run_field(_multi)'s host path
    e2e = None
    if not args.no_e2e:
        nfield = ncell * (len(w.thetas) if multi_fields is not None and not args.separate_iso and not args.dense else 1)
        Xh = torch.from_numpy(np.array(w.X)).pin_memory().numpy()
        yh = torch.from_numpy(np.array(w.y)).pin_memory().numpy()
        fh = torch.empty(nfield, dtype=torch.float32).pin_memory().numpy()
        host = (Xh, yh, fh)
        step(host)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        leaves_e = 0
        for _ in range(args.e2e_steps):
            leaves_e += step(host)[0]
        torch.cuda.synchronize()
        barrier()
        te = torch.tensor([(time.perf_counter() - t0) / args.e2e_steps, leaves_e / args.e2e_steps],
                          dtype=torch.float64, device=dev)
        if world > 1:
            tl = te.clone()
            all_reduce(te, dist.ReduceOp.MAX)
            all_reduce(tl, dist.ReduceOp.SUM)
            te[1] = tl[1]
        e2e = {"value": float(te[1]) / float(te[0]), "unit": UNIT,
               "h2d_bytes_per_step": int(Xh.nbytes + yh.nbytes),
               "d2h_bytes_per_step": int(fh.nbytes) * (1 if len(w.thetas) == 1 or fh.size > ncell else len(w.thetas)),
               "seconds_per_step": float(te[0]),
               "path": ("C ABI host pointers: lcp_fit_local(xy_on_device=0), lcp_run_field(_multi)(out_on_device=0)"
                        if world == 1 else "lcp_fit_local host inputs; slab fields gathered to rank 0, then read back")}

    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return 0
    # roofline of the dominant kernel (k_pmc): algorithmic lane-ops / measured time
    mc_s = float(t[1]) / args.steps / 1000.0
    peak = SM_COUNT * LANES_PER_SM_CLK * 1965e6 / 1e12          # T lane-op/s at the max SM clock
    p2_step = float(lv[2]) / args.steps
    fused_t = len(w.thetas) if len(w.thetas) > 1 and not args.dense and not args.separate_iso else 1
    ops_step = (samples_step * (OPS_PHASE1 + OPS_PHASE1_PER_EXTRA_ISO * (fused_t - 1))
                + p2_step * (OPS_PHASE2 + OPS_PHASE2_PER_EXTRA_ISO * (fused_t - 1)))
    impl_mix = (ops_step / max(world, 1)) / mc_s / 1e12 if mc_s > 0 else None
    ops_survey = samples_step * (OPS_SURVEY + OPS_SURVEY_PER_EXTRA_ISO * (fused_t - 1))
    achieved = (ops_survey / max(world, 1)) / mc_s / 1e12 if mc_s > 0 else None
    launches_per_step = 1 if fused_t > 1 else len(w.thetas)      # k_pmc launches per step
    traffic = load_traffic(union_step / max(world, 1) / launches_per_step)
    roofline = {"bound": "alu", "kernel": "k_pmc", "achieved": achieved, "peak": peak,
                "unit": "Tlane-op/s", "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "ops_per_sample": ops_survey / samples_step if samples_step else None,
                "ops_note": ("achieved = samples x SURVEY.md 8(d) minimal op mix (186 issue slots per "
                             "sample, +21 per extra fused isovalue) / summed k_pmc time; the two-phase "
                             "kernel executes fewer: frac_impl_mix uses its own fixed mix (106 per "
                             "sample + 93 per phase-2 sample)"),
                "frac_impl_mix": (impl_mix / peak) if impl_mix else None,
                "impl_ops_per_sample": ops_step / samples_step if samples_step else None,
                "phase2_fraction": p2_step / samples_step if samples_step else None,
                "samples_per_s": samples_step / max(world, 1) / mc_s if mc_s > 0 else None,
                "mc_share_of_step": mc_s / (ms_step / 1000.0),
                # plain FP32 FLOP/s of the same kernel (FMA = 2): per sample
                # 26 FMA of the partial L'z, 4 of the bounds, 2 x (angle FMA + 2 products + uniform
                # add) of Box-Muller = 70 flop; per phase-2 sample 10 FMA + 4 adds + 10 = 34 flop
                "fp32_tflops": ((samples_step * 70 + p2_step * 34) / max(world, 1) / mc_s / 1e12
                                if mc_s > 0 else None),
                "fp32_peak_tflops": 74.4,
                "hbm": hbm_fractions(union_step / max(world, 1) / launches_per_step, mc_s / launches_per_step),
                "peak_note": "148 SMs x 128 lanes x 1.965 GHz issue slots (guide unit counts, max clock)"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            import oracle as O
            v, secs, detail = oracle_sample(w, 1, 0)
            cpu = {"value": v, "unit": UNIT, "cores": O.num_threads(), "kind": "oracle",
                   "sample": detail["sample"], "measured_s": secs + detail["model_build_s"],
                   "extrapolated_full_workload_s": detail["extrapolated_full_workload_s"]}
        except Exception as ex:  # the GPU number stands on its own
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"failed: {ex}"}
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64/f32", "data": "synthetic",
           "config": {"workload": workload_desc(cfg, w.thetas) + (
                          f" | DENSE baseline ({args.dense} GP), every cell" if args.dense else ""),
                      "mode": f"dense-{args.dense}" if args.dense else "octree-pruned",
                      "isovalue_pass": ("fused multi-isovalue leaf pass (NEXT-3)" if len(w.thetas) > 1 and not
                                        args.dense and not args.separate_iso else "one pass per isovalue"), "extreme_iters": args.extreme, "cells": ncell, "m": cfg.m, "k": k,
                      "n_samples": cfg.n_samples, "alpha": cfg.alpha, "max_depth": cfg.max_depth,
                      "parallelism": f"z-slab x{world}" if world > 1 else "single GPU",
                      "l2": "flushed between timed steps (256 MB write, outside the step events)"},
           "end_to_end_octree_lcp_s": ms_step / 1000.0,
           "leaf_cells_per_step": leaves_step, "grid_cells_per_s": cells_per_step / (ms_step / 1000.0),
           "pmc_cells_per_step": union_step,
           "samples_per_step": samples_step,
           "phase_ms_per_step": {k2: v2 / args.steps for k2, v2 in st_phase.items()},
           "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(float(lv[1])),
           "paper_context": PAPER_CONTEXT,
           "clocks": clk}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
