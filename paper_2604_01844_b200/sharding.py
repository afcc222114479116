"""Multi-GPU decomposition of the two hot paths.

* Rasterizer — view sharding: rank r owns views {v : v mod P == r}; every rank holds the
  full cloud, sums its views' gradients in fp64 (gsct_rasterize_bwd does the per-rank view
  sum), then one all-reduce (sum) of the packed gradient buffer and one (max) of the
  visibility bytes. Images stay rank-local. Oracle: sum over all views of
  rasterize_backward via ParamGradients::add (core.hpp:152-162).
* Voxelizer — z-slab sharding: rank r owns the r-th of P contiguous z-slabs. Forward needs no
  communication (each rank writes its slab; boxes are computed in full-grid coordinates,
  so slabs tile the full-grid volume bit for bit). Backward: per-splat moment partial
  sums over the slab, fp64 all-reduce (sum) of the [10, N] moments, then the fp64 finish.
  pos_grad_norm is formed after the reduction (the norm is nonlinear).

The functions take a `torch.distributed` process group (NCCL on GPUs; gloo in the CPU
tests) and only move data that the path must exchange. `native_group` instead builds the
library's own group (include/gsct_cuda.h, multi-GPU): one NCCL communicator per context,
whose reductions the C-ABI calls enqueue themselves -- the path a C++ caller of the
reference API takes.
"""
from __future__ import annotations

from typing import Sequence


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """Views owned by `rank` (round-robin, so ranks get 10/9 of 75 views at P = 8)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_views: bad rank/world")
    return list(range(rank, n_views, world))


def zslab_windows(dims: Sequence[int], world: int) -> list[tuple[tuple[int, int, int], tuple[int, int, int]]]:
    """[lo, hi) windows of equal z-slabs (the first nz % P slabs one slice thicker)."""
    nx, ny, nz = (int(d) for d in dims)
    if world < 1:
        raise ValueError("zslab_windows: world must be >= 1")
    out = []
    base, extra = divmod(nz, world)
    z = 0
    for r in range(world):
        dz = base + (1 if r < extra else 0)
        out.append(((0, 0, z), (nx, ny, z + dz)))
        z += dz
    return out


def pack_grads(n: int, like=None):
    """One flat fp64 buffer [12N] with ParamGradients views into it (single all-reduce):
    positions [0,3N), log_scales [3N,6N), rotations [6N,10N), raw_densities, pos_grad_norm."""
    import torch

    from .gsct import ParamGradients

    dev = like.device if like is not None else "cpu"
    flat = torch.zeros(12 * n, dtype=torch.float64, device=dev)
    g = ParamGradients(flat[0:3 * n].view(n, 3), flat[3 * n:6 * n].view(n, 3), flat[6 * n:10 * n].view(n, 4),
                       flat[10 * n:11 * n], flat[11 * n:12 * n], torch.zeros(n, dtype=torch.uint8, device=dev))
    return flat, g


def allreduce_grads(flat, visible, group=None) -> None:
    """Sum the packed per-rank view sums; OR the visibility bytes (as max)."""
    import torch.distributed as dist

    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(visible, op=dist.ReduceOp.MAX, group=group)


def native_group(ctx, pg=None):
    """The library's NCCL group over the ranks of `pg` (default: the world), attached to
    `ctx`: rank 0 makes the id, a torch.distributed broadcast hands it to every rank."""
    import torch.distributed as dist

    rank, world = dist.get_rank(pg), dist.get_world_size(pg)
    box = [ctx.group_new_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(pg, 0) if pg is not None else 0, group=pg)
    return ctx.create_group(box[0], world, rank, attach=True)


def allreduce_moments(moments, group=None) -> None:
    """Sum the [10, N] fp64 voxel-backward partial moments over the z-slabs."""
    import torch.distributed as dist

    dist.all_reduce(moments, op=dist.ReduceOp.SUM, group=group)
