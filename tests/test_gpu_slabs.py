"""The N > 1 path of SURVEY §8(e) on the GPU: z-slab contexts with the automatic
slab level and weighted cuts, slab-local MC record tables, and the gather to
rank 0.  The rank-0 field equals the single-GPU field bit for bit (Philox keyed
by the global cell id; node decisions are local to the node)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from workloads import generate

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name,world,shard", [("c2", 2, False), ("c2", 8, False), ("c4", 2, False),
                                              ("c4", 8, False), ("c5", 8, False), ("c2", 3, True), ("c4", 8, True),
                                              ("c1", 8, True)])
def test_torchrun_gather_equals_single_gpu(name, world, shard, tmp_path):
    # shard: the bucket factors split across the ranks and all-gathered (dist.fit_sharded)
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tools", "dist_check.py"),
           "--workload", name, "--out", str(out)] + (["--fit-shard"] if shard else [])
    env = dict(os.environ, OMP_NUM_THREADS="1")
    p = subprocess.run(cmd, cwd=ROOT, env=env, timeout=1200, capture_output=True, text=True)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    res = json.load(open(out))
    print(json.dumps({k: res[k] for k in ("workload", "world", "slab_level", "layers", "layer_cuts",
                                          "leaves_per_rank", "record_cells_per_rank")}))
    assert res["bitexact"], res["max_abs_diff"]
    assert res["leaves_sum"] == res["leaves_n1"]
    # no empty rank (c1: 16^3 cells, 2 slab layers for 8 ranks -- more ranks than layers, and
    # more ranks than buckets for the sharded fit), the same plan on every rank
    if name != "c1":
        assert all(sum(lv) > 0 for lv in res["leaves_per_rank"]), res["leaves_per_rank"]
    assert all(c == res["layer_cuts"][0] for c in res["layer_cuts"])
    assert len(res["layer_cuts"][0]) == world + 1
    # slab-local record tables, used by every rank's leaf pass
    if res["records_used_n1"]:
        used = [u for u, lv in zip(res["records_used_per_rank"], res["leaves_per_rank"]) if sum(lv) > 0]
        assert all(used), res["records_used_per_rank"]
        lf = {"c1": 4, "c2": 6, "c4": 8, "c5": 9}[name]
        assert max(res["record_cells_per_rank"]) < (1 << (3 * lf))   # slab-local: below the whole cube


@pytest.mark.parametrize("name,G", [("p1", 4), ("c3", 3), ("t2", 2)])
def test_auto_slabs_union_equals_full(name, G, dev):
    # ranks run one after another on one GPU: automatic level, weighted cuts
    from paper_2512_12442_b200 import Context, config_args
    w = generate(name)
    cfg = w.cfg
    kernel, grid, k, b, hf = config_args(cfg)
    X = torch.from_numpy(np.array(w.X)).to(dev)
    y = torch.from_numpy(np.array(w.y)).to(dev)
    th = w.thetas[0]
    full = Context(0).fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf)
    ref, n_ref = full.run_field(th, cfg.alpha, cfg.max_depth, cfg.n_samples, cfg.mc_seed)
    ref = ref.clone()
    acc = torch.zeros_like(ref)
    counts, cuts = [], []
    for r in range(G):
        ctx = Context(0).fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf, slab_rank=r, slab_count=G)
        f, n = ctx.run_field(th, cfg.alpha, cfg.max_depth, cfg.n_samples, cfg.mc_seed)
        st = ctx.stats()
        acc += f
        counts.append(n)
        cuts.append(st["slab"]["layer_cuts"])
        # a second refine of the same fit keeps the plan (records stay valid)
        f2, n2 = ctx.run_field(th, cfg.alpha, cfg.max_depth, cfg.n_samples, cfg.mc_seed)
        assert n2 == n and torch.equal(f2, f)
    assert torch.equal(acc, ref)
    assert sum(counts) == n_ref
    assert all(c == cuts[0] for c in cuts)
    if name != "t2":
        assert min(counts) > 0, counts
    print(name, G, "leaves per rank", counts, "max/mean", max(counts) / (sum(counts) / G))


def test_slab_refine_shallower_than_plan(dev):
    # a refine whose max_depth stops above the planned slab level still partitions the
    # cells (leaf cells filtered by z), and a later full-depth refine keeps the plan
    from paper_2512_12442_b200 import Context, config_args
    w = generate("c2")
    cfg = w.cfg
    kernel, grid, k, b, hf = config_args(cfg)
    X = torch.from_numpy(np.array(w.X)).to(dev)
    y = torch.from_numpy(np.array(w.y)).to(dev)
    th = w.thetas[0]
    full = Context(0).fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf)
    G = 3
    for depth in (cfg.max_depth, 1, cfg.max_depth):
        ref = np.sort(full.octree_refine(th, cfg.alpha, depth).cpu().numpy())
        parts = []
        for r in range(G):
            ctx = Context(0).fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf, slab_rank=r, slab_count=G)
            ctx.octree_refine(th, cfg.alpha, cfg.max_depth)          # places the plan
            parts.append(ctx.octree_refine(th, cfg.alpha, depth).cpu().numpy())
        allp = np.concatenate(parts)
        assert len(allp) == len(np.unique(allp))
        assert np.array_equal(np.sort(allp), ref), depth


def test_sharded_fit_state_machine(dev):
    # lcp_fit_shard_buffers / lcp_fit_finish only while a sharded fit is pending; every other
    # call returns ESTATE in between; an unsharded fit has nothing pending
    from paper_2512_12442_b200 import Context, LcpError, config_args
    from paper_2512_12442_b200.lcp import LCP_ESTATE
    w = generate("t2")
    cfg = w.cfg
    kernel, grid, k, b, hf = config_args(cfg)
    ctx = Context(0).fit_local(w.X, w.y, kernel, k, grid, bucket_log2=b, h_full=hf)
    for call in (ctx.fit_shard_buffers, ctx.fit_finish):
        with pytest.raises(LcpError) as e:
            call()
        assert e.value.status == LCP_ESTATE
    ctx.fit_local(w.X, w.y, kernel, k, grid, bucket_log2=b, h_full=hf, slab_rank=0, slab_count=2, fit_shard=1)
    with pytest.raises(LcpError) as e:
        ctx.octree_refine(w.thetas[0], cfg.alpha, cfg.max_depth)
    assert e.value.status == LCP_ESTATE
    bd, nb, sets, ns = ctx.fit_shard_buffers()
    assert bd.numel() == 2 * nb and sets.numel() == 2 * ns
    # stand-in for the other rank's chunk: a second context's own sharded fit
    other = Context(0).fit_local(w.X, w.y, kernel, k, grid, bucket_log2=b, h_full=hf, slab_rank=1, slab_count=2,
                                 fit_shard=1)
    obd, _, osets, _ = other.fit_shard_buffers()
    bd[nb:].copy_(obd[nb:])
    sets[ns:].copy_(osets[ns:])
    ctx.fit_finish()
    with pytest.raises(LcpError):
        ctx.fit_finish()
    # the completed model equals an unsharded one (same refine, same slab plan)
    ref = Context(0).fit_local(w.X, w.y, kernel, k, grid, bucket_log2=b, h_full=hf, slab_rank=0, slab_count=2)
    a = ctx.run_field(w.thetas[0], cfg.alpha, cfg.max_depth, 500, 3)[0]
    r = ref.run_field(w.thetas[0], cfg.alpha, cfg.max_depth, 500, 3)[0]
    assert torch.equal(a, r)
    assert torch.equal(ctx.bucket_sets(), ref.bucket_sets())
