"""Multi-process (world_size 2 and 3, gloo, CPU) tests of the z-slab host logic:
the slab partition tiles the grid, and gather_field assembles rank slices on
rank 0 exactly.  The GPU-side slab filter is checked against
the single-domain run in tests/test_gpu_parity.py::test_slab_union_equals_full."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_12442_b200.dist import gather_field, lfull_of, min_slab_level, slab_cells, slab_layers


@pytest.mark.parametrize("cells", [(16, 16, 16), (23, 17, 11), (40, 9, 33), (512, 512, 512), (256, 256, 128)])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_slab_partition_tiles_grid(cells, world):
    lvl = max(min_slab_level(world), 3) if lfull_of(cells) >= 3 else min_slab_level(world)
    lvl = min(lvl, lfull_of(cells))
    covered = []
    for r in range(world):
        z0, z1 = slab_layers(cells, lvl, r, world)
        assert z0 <= z1
        covered.append(slab_cells(cells, lvl, r, world))
    assert covered[0][0] == 0
    assert covered[-1][1] == cells[0] * cells[1] * cells[2]
    for (a0, a1), (b0, b1) in zip(covered, covered[1:]):
        assert a1 == b0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cells, lvl, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = cells[0] * cells[1] * cells[2]
    field = torch.zeros(n)
    c0, c1 = slab_cells(cells, lvl, rank, world)
    field[c0:c1] = torch.arange(c0, c1, dtype=torch.float32) * 0.5 + rank * 1e-3
    out = gather_field(field, cells, lvl)
    if rank == 0:
        want = torch.zeros(n)
        for r in range(world):
            a, b = slab_cells(cells, lvl, r, world)
            want[a:b] = torch.arange(a, b, dtype=torch.float32) * 0.5 + r * 1e-3
        q.put(bool(torch.equal(out, want)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cells", [(16, 16, 16), (23, 17, 11)])
def test_gather_field_gloo(world, cells):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    lvl = min(3, lfull_of(cells))
    procs = [ctx.Process(target=_worker, args=(r, world, port, cells, lvl, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok
