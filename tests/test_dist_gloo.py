"""Host logic of the z-slab decomposition, on the CPU:

* the slab plan liblcp's refine applies (lcp_slab_auto_level / lcp_slab_cuts,
  host-only C ABI calls): the automatic level gives every rank >= 1 z-layer, the
  weighted cuts tile the layers contiguously and minimise the largest rank weight
  (brute force on small cases), within one layer of the ideal;
* gather_fields assembles the ranks' slab slices (uneven, several isovalue rows)
  on rank 0 exactly -- multi-process, world_size 2 and 3, gloo.

The GPU-side slab filter is checked against the single-domain run bit for bit in
tests/test_gpu_parity.py (test_slab_union_equals_full*)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_12442_b200.dist import (_allgather_inplace, cell_ranges, cell_z_cuts, equal_z_cuts, gather_fields,
                                        layers_at, lfull_of)
from paper_2512_12442_b200.lcp import slab_auto_level, slab_cuts

GRIDS = [(16, 16, 16), (23, 17, 11), (40, 9, 33), (64, 64, 64), (128, 128, 128), (256, 256, 128), (512, 512, 512),
         (1024, 1024, 1024)]


@pytest.mark.parametrize("cells", GRIDS)
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_auto_level_gives_every_rank_a_layer(cells, world):
    lf = lfull_of(cells)
    lv = slab_auto_level(cells, world, lf)
    assert 1 <= lv <= max(1, lf - 3)
    nz = layers_at(cells, lv)
    if lf >= 4 and layers_at(cells, max(1, lf - 3)) >= world:
        assert nz >= world, (cells, world, lv, nz)
    if lv > 1:
        assert layers_at(cells, lv - 1) < 2 * world     # the shallowest such level
    # capped by max_depth
    assert slab_auto_level(cells, world, 1) == 1


def _loads(w, cuts):
    P = np.concatenate([[0], np.cumsum(w)])
    return np.array([P[cuts[r + 1]] - P[cuts[r]] for r in range(len(cuts) - 1)])


@pytest.mark.parametrize("world", [2, 3, 4, 5, 8])
def test_weighted_cuts_tile_and_balance(world):
    g = np.random.default_rng(world)
    for trial in range(40):
        nz = int(g.integers(world, 14 if trial % 2 else 80))
        kind = trial % 4
        if kind == 0:
            w = g.integers(0, 1000, nz)
        elif kind == 1:   # thin shell: a few heavy layers
            w = np.zeros(nz, np.int64)
            w[g.choice(nz, min(nz, 3), replace=False)] = g.integers(100, 5000, min(nz, 3))
        elif kind == 2:   # ramp
            w = np.arange(nz) * 7 + 1
        else:             # dense c5-like: all equal
            w = np.full(nz, 1024)
        cuts = slab_cuts(w, world)
        assert cuts[0] == 0 and cuts[-1] == nz
        assert np.all(np.diff(cuts) >= 1), (w, cuts)          # every rank >= 1 layer (nz >= world)
        loads = _loads(w, cuts)
        assert loads.sum() == w.sum()
        # the largest rank weight exceeds the ideal by less than one layer
        assert loads.max() <= w.sum() / world + w.max() + 1e-9, (w, cuts, loads)
        # and is optimal over all contiguous cuts (brute force on small cases)
        if nz <= 14 and world <= 4:
            import itertools
            best = min(_loads(w, (0,) + c + (nz,)).max()
                       for c in itertools.combinations(range(1, nz), world - 1))
            assert loads.max() == best, (w, cuts, loads, best)


def test_cuts_zero_weights_and_more_ranks_than_layers():
    assert list(slab_cuts([0] * 8, 4)) == [0, 2, 4, 6, 8]
    c = slab_cuts([5, 1, 9], 5)         # fewer layers than ranks: some ranks get none
    assert c[0] == 0 and c[-1] == 3 and np.all(np.diff(c) >= 0)
    with pytest.raises(Exception):
        slab_cuts([1, -1, 2], 2)


@pytest.mark.parametrize("cells", GRIDS)
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_equal_plan_tiles_grid(cells, world):
    zc = equal_z_cuts(cells, world, lfull_of(cells))
    rng = cell_ranges(cells, zc)
    assert rng[0][0] == 0 and rng[-1][1] == cells[0] * cells[1] * cells[2]
    for (a0, a1), (b0, b1) in zip(rng, rng[1:]):
        assert a1 == b0 and a0 <= a1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cells, zc, T, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = cells[0] * cells[1] * cells[2]
    rng = cell_ranges(cells, zc)
    fields = torch.zeros((T, n))
    c0, c1 = rng[rank]
    for t in range(T):
        fields[t, c0:c1] = torch.arange(c0, c1, dtype=torch.float32) * 0.5 + rank * 1e-3 + t
    out = gather_fields(fields if T > 1 else fields[0], cells, zc)
    if rank == 0:
        want = torch.zeros((T, n))
        for r in range(world):
            a, b = rng[r]
            for t in range(T):
                want[t, a:b] = torch.arange(a, b, dtype=torch.float32) * 0.5 + r * 1e-3 + t
        q.put(bool(torch.equal(out.view(T, n), want)))
    else:
        # only rank 0 receives: the other ranks' fields are untouched
        q.put(bool(torch.count_nonzero(fields[:, :c0]) == 0 and torch.count_nonzero(fields[:, c1:]) == 0))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cells,T", [((16, 16, 16), 1), ((23, 17, 11), 3), ((40, 9, 33), 2)])
def test_gather_fields_gloo(world, cells, T):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    lv = slab_auto_level(cells, world, lfull_of(cells))
    nz = layers_at(cells, lv)
    w = np.random.default_rng(nz + world).integers(0, 50, nz)
    zc = cell_z_cuts(cells, lv, slab_cuts(w, world))
    procs = [ctx.Process(target=_worker, args=(r, world, port, cells, zc, T, q)) for r in range(world)]
    for p in procs:
        p.start()
    oks = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(oks)


def _ag_worker(rank, world, port, chunk, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    buf = torch.zeros(world * chunk, dtype=torch.uint8)
    buf[rank * chunk:(rank + 1) * chunk] = torch.arange(chunk, dtype=torch.int64).remainder(251).to(torch.uint8) + rank
    _allgather_inplace(buf, chunk)
    want = torch.cat([torch.arange(chunk, dtype=torch.int64).remainder(251).to(torch.uint8) + r for r in range(world)])
    q.put(bool(torch.equal(buf, want)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fit_allgather_gloo(world):
    # the in-place all-gather of dist.fit_sharded: rank r's chunk of the ctx-owned bucket
    # blocks is sent, the others' are received in place
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ag_worker, args=(r, world, port, 1000 + 7 * world, q)) for r in range(world)]
    for p in procs:
        p.start()
    oks = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(oks)
