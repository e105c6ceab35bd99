#!/usr/bin/env python
"""Functional check of the N > 1 path on however many GPUs exist:
launched under torch.distributed.run, every rank fits its z-slab context, runs the
bench step (lcp_run_field, or the fused lcp_run_field_multi for several
isovalues) and the fields are gathered to rank 0 (dist.gather_fields), which
compares them bit for bit with a single-domain (N = 1) run of its own.

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \
        tools/dist_check.py --workload c4 --out result.json

With fewer GPUs than ranks the ranks share devices round-robin and the
collectives run over gloo (host copies); the partition, the slab filter, the
slab-local record tables and the gather are the ones a multi-GPU run uses.
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
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--out", required=True)
    ap.add_argument("--n-samples", type=int, default=0, help="override N (0 = the config's)")
    ap.add_argument("--fit-shard", action="store_true", help="shard the bucket factors (dist.fit_sharded)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2512_12442_b200 import Context, config_args
    from paper_2512_12442_b200.dist import fit_sharded, gather_fields, plan_z_cuts
    from workloads import generate

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    ngpu = torch.cuda.device_count()
    local = int(os.environ.get("LOCAL_RANK", "0")) % ngpu
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    backend = "nccl" if ngpu >= world else "gloo"
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    dist.barrier()
    w = generate(args.workload)
    cfg = w.cfg
    N = args.n_samples or cfg.n_samples
    kernel, grid, k, b, hf = config_args(cfg)
    X = torch.from_numpy(np.array(w.X)).to(dev)
    y = torch.from_numpy(np.array(w.y)).to(dev)
    ncell = int(np.prod(cfg.cells))
    T = len(w.thetas)
    # the single-GPU reference first (rank 0), kept on the host, its context freed before the
    # slab contexts are built: all ranks may share one device
    ref, nl_ref, full_records = None, None, None
    if rank == 0:
        ref_ctx = Context(local).fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf)
        if T > 1:
            r_, nl_r, _ = ref_ctx.run_field_multi(list(w.thetas), cfg.alpha, cfg.max_depth, N, cfg.mc_seed, 0)
            nl_ref = [int(v) for v in nl_r]
        else:
            r_, n_r = ref_ctx.run_field(w.thetas[0], cfg.alpha, cfg.max_depth, N, cfg.mc_seed)
            r_, nl_ref = r_.view(1, -1), [int(n_r)]
        ref = r_.cpu()
        full_records = ref_ctx.stats()["pmc_used_records"]
        del r_, ref_ctx
        torch.cuda.empty_cache()
    dist.barrier()
    if args.fit_shard:
        ctx = fit_sharded(Context(local), X, y, kernel, k, grid, rank, world, bucket_log2=b, h_full=hf)
    else:
        ctx = Context(local).fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf, slab_rank=rank,
                                       slab_count=world)
    if T > 1:
        fields, nl, nu = ctx.run_field_multi(list(w.thetas), cfg.alpha, cfg.max_depth, N, cfg.mc_seed, 0)
        nleaf = [int(v) for v in nl]
    else:
        f, n = ctx.run_field(w.thetas[0], cfg.alpha, cfg.max_depth, N, cfg.mc_seed)
        fields = f.view(1, -1)
        nleaf = [int(n)]
    st = ctx.stats()
    zc = plan_z_cuts(st)
    gather_fields(fields, cfg.cells, zc)
    torch.cuda.synchronize()
    info = {"rank": rank, "leaves": nleaf, "slab": st["slab"], "pmc_used_records": st["pmc_used_records"],
            "fused": st["fused"]}
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(info, gathered, dst=0)
    if rank == 0:
        got = fields.cpu()
        res = {"workload": args.workload, "world": world, "backend": backend, "gpus": ngpu,
               "fit_shard": bool(args.fit_shard),
               "bitexact": bool(torch.equal(got, ref)),
               "max_abs_diff": float((got - ref).abs().max()),
               "leaves_n1": nl_ref, "leaves_per_rank": [g["leaves"] for g in gathered],
               "leaves_sum": [int(sum(g["leaves"][t] for g in gathered)) for t in range(T)],
               "layer_cuts": [g["slab"]["layer_cuts"] for g in gathered],
               "slab_level": gathered[0]["slab"]["level"], "layers": gathered[0]["slab"]["layers"],
               "weights": gathered[0]["slab"]["weights"],
               "record_cells_per_rank": [g["slab"]["record_cells"] for g in gathered],
               "records_used_per_rank": [g["pmc_used_records"] for g in gathered],
               "records_used_n1": full_records, "ncell": ncell}
        json.dump(res, open(args.out, "w"))
        print(json.dumps(res))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
