"""z-slab decomposition of the octree across GPUs.

Every rank holds the same bucket-local GP (observations replicated: the halo;
with `fit_sharded` each rank factors 1/N of the buckets and the blocks are
all-gathered in place), refines octree levels 0 .. slab_level redundantly, and the first refine after
the fit cuts the z-layers of level `slab_level` into contiguous per-rank ranges
by prefix sums of the refined nodes per layer -- computed identically on every
rank, so no communication is needed (liblcp, octree.cu).  Each rank then
finishes refine + PMC on its own subtrees.  Results are bit-identical to one GPU:
Philox counters are keyed by the global cell id and every node decision is local
to the node.  The collectives: the all-gather of the sharded bucket factors
after the fit, and the final gather of the per-slab slices of the dense field(s)
to rank 0 (point-to-point: only rank 0 receives).

This module is plumbing only (range arithmetic and torch.distributed calls); the
slab plan itself is liblcp's (lcp_slab_auto_level / lcp_slab_cuts, host-only).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

from .lcp import slab_auto_level, slab_cuts


def lfull_of(cells) -> int:
    cmax = max(cells)
    lf = 0
    while (1 << lf) < cmax:
        lf += 1
    return lf


def layers_at(cells, level: int) -> int:
    side = 1 << (lfull_of(cells) - level)
    return (cells[2] + side - 1) // side


def cell_z_cuts(cells, level: int, layer_cuts: Sequence[int]) -> List[int]:
    """Layer cuts of `level` -> cut z-planes of cells (clipped to the grid)."""
    side = 1 << (lfull_of(cells) - level)
    return [min(int(z) * side, cells[2]) for z in layer_cuts]


def cell_ranges(cells, z_cuts: Sequence[int]) -> List[Tuple[int, int]]:
    """Per-rank [c0, c1) ranges of linear cell ids (x fastest): rank r's slab is the
    z-planes [z_cuts[r], z_cuts[r + 1])."""
    plane = cells[0] * cells[1]
    return [(int(z_cuts[r]) * plane, int(z_cuts[r + 1]) * plane) for r in range(len(z_cuts) - 1)]


def equal_z_cuts(cells, world: int, max_depth: int) -> List[int]:
    """Unweighted plan (the dense baseline, which has no octree): equal layer counts at
    the automatic slab level."""
    lv = slab_auto_level(cells, world, max_depth)
    return cell_z_cuts(cells, lv, slab_cuts([0] * layers_at(cells, lv), world))


def plan_z_cuts(stats: dict) -> List[int]:
    """The z-plane cuts of the slab plan a context reports (lcp_stats_json "slab")."""
    return list(stats["slab"]["cell_z_cuts"])


def gather_fields(fields, cells, z_cuts: Sequence[int], group=None):
    """Assemble the dense LCP field(s) on rank 0 from the ranks' slab slices.

    `fields` is this rank's (T, nx*ny*nz) (or flat) field tensor, zero outside its
    slab.  Every rank r > 0 sends its T contiguous slices [c0_r, c1_r) to rank 0, which
    receives them in place (one batch of point-to-point transfers; the other ranks
    receive nothing).  Returns `fields` (complete on rank 0)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return fields
    rows = fields.view(1, -1) if fields.dim() == 1 else fields
    ranges = cell_ranges(cells, z_cuts)
    gloo = dist.get_backend(group) == "gloo"      # gloo moves host tensors only
    ops, staged = [], []
    if rank == 0:
        for r in range(1, world):
            a, b = ranges[r]
            if b <= a:
                continue
            for t in range(rows.shape[0]):
                buf = torch.empty(b - a, dtype=rows.dtype) if gloo else rows[t, a:b]
                ops.append(dist.P2POp(dist.irecv, buf, r, group))
                staged.append((t, a, b, buf))
    else:
        a, b = ranges[rank]
        if b > a:
            for t in range(rows.shape[0]):
                buf = rows[t, a:b].cpu() if gloo else rows[t, a:b]
                ops.append(dist.P2POp(dist.isend, buf, 0, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if rank == 0 and gloo:
        for t, a, b, buf in staged:
            rows[t, a:b] = buf.to(rows.device)
    return fields


def _allgather_inplace(buf, chunk: int, group=None):
    """All-gather, in place, the equal byte chunks of a uint8 CUDA tensor: rank r's chunk
    buf[r chunk:(r + 1) chunk] is sent, every other chunk is received."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    if dist.get_backend(group) == "gloo":          # gloo moves host tensors only
        out = torch.empty(buf.numel(), dtype=torch.uint8)
        dist.all_gather_into_tensor(out, buf[rank * chunk:(rank + 1) * chunk].cpu(), group=group)
        buf.copy_(out)                             # host -> device, no device temporary
    else:
        send = buf[rank * chunk:(rank + 1) * chunk].clone()
        dist.all_gather_into_tensor(buf, send, group=group)
        del send


def fit_sharded(ctx, xyz, y, kernel, k, grid, slab_rank: int, slab_count: int, group=None, **kw):
    """lcp_fit_local with the bucket work split across the ranks (opts.fit_shard): each rank
    computes the local sets and factors of 1/slab_count of the buckets, the blocks are
    all-gathered in place (one NCCL all-gather; c5: 2.3 GB of factors), and lcp_fit_finish
    computes the observation marginals.  Identical model to an unsharded fit, bit for bit."""
    ctx.fit_local(xyz, y, kernel, k, grid, slab_rank=slab_rank, slab_count=slab_count, fit_shard=1, **kw)
    bdata, nb, sets, ns = ctx.fit_shard_buffers()
    _allgather_inplace(bdata, nb, group)
    _allgather_inplace(sets, ns, group)
    return ctx.fit_finish()


def gather_field(field, cells, z_cuts: Sequence[int], group=None):
    """One field (flat): see gather_fields."""
    return gather_fields(field, cells, z_cuts, group)
