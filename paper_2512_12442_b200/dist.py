"""z-slab decomposition of the octree across GPUs.

Every rank fits the same bucket-local GP (observations replicated: the halo),
refines octree levels 0 .. slab_level-1 redundantly, then keeps only the
level-`slab_level` nodes whose z index lies in its slab (the filter is applied
inside liblcp, k_node_counts / k_emit) and finishes refine + PMC on its own
subtrees.  Results are bit-identical to one GPU: Philox counters are keyed by
the global cell id and every node decision is local to the node.  The only
collective is the final gather of the per-slab dense-field slices to rank 0.

This module is plumbing only (partition arithmetic and torch.distributed
calls); all LCP arithmetic runs in liblcp.so.
"""
from __future__ import annotations

from typing import Tuple


def lfull_of(cells) -> int:
    cmax = max(cells)
    lf = 0
    while (1 << lf) < cmax:
        lf += 1
    return lf


def slab_layers(cells, slab_level: int, rank: int, world: int) -> Tuple[int, int]:
    """z range [z0, z1) of level-`slab_level` nodes owned by `rank` (same rule
    as liblcp's refine: equal split of the node layers that hold cells)."""
    lf = lfull_of(cells)
    side = 1 << (lf - slab_level)
    nz = (cells[2] + side - 1) // side
    return rank * nz // world, (rank + 1) * nz // world


def slab_cells(cells, slab_level: int, rank: int, world: int) -> Tuple[int, int]:
    """[c0, c1) range of linear cell ids (x fastest) covered by the rank's slab:
    its cells are exactly the z-planes [z0 * side, min(z1 * side, nz))."""
    lf = lfull_of(cells)
    side = 1 << (lf - slab_level)
    z0, z1 = slab_layers(cells, slab_level, rank, world)
    plane = cells[0] * cells[1]
    return min(z0 * side, cells[2]) * plane, min(z1 * side, cells[2]) * plane


def min_slab_level(world: int) -> int:
    lvl = 0
    while (1 << lvl) < world:
        lvl += 1
    return max(lvl, 1)


def gather_field(field, cells, slab_level: int, group=None):
    """Assemble the dense LCP field on rank 0 from the ranks' slab slices.

    `field` is this rank's full-size flat field (zeros outside its slab).  Each
    rank contributes only its contiguous slab slice (padded to the largest
    slab); rank 0 receives them with one all_gather_into_tensor and writes them
    in place.  Returns the assembled field on rank 0 (other ranks: their input).
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return field
    ranges = [slab_cells(cells, slab_level, r, world) for r in range(world)]
    width = max(c1 - c0 for c0, c1 in ranges)
    c0, c1 = ranges[rank]
    # gloo moves host tensors only: stage CUDA slices through the host
    dev = "cpu" if dist.get_backend(group) == "gloo" else field.device
    send = torch.zeros(width, dtype=field.dtype, device=dev)
    send[: c1 - c0] = field[c0:c1]
    recv = torch.empty(world * width, dtype=field.dtype, device=dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    if rank == 0:
        for r, (a, b) in enumerate(ranges):
            field[a:b] = recv[r * width: r * width + (b - a)]
    return field
