"""Multi-GPU path through the boundary (SURVEY.md 8(b) gsct_group, 8(e)), on the one-GPU box.

* The library's own group (include/gsct_cuda.h, multi-GPU: one NCCL communicator per
  context) at world size 1: the grouped backward / voxel calls (all-reduce on the context
  stream, slab all-gather) give results bit-identical to the ungrouped calls.
* World size 2 with the CUDA operators per rank (two processes sharing cuda:0; NCCL refuses
  two ranks on one device, so the exchange is gloo): round-robin view shards of
  gsct_rasterize_bwd summed across ranks equal the oracle's sum over all views of
  rasterize_backward (ParamGradients::add, core.hpp:152-162) within 1e-4 per class; z-slab
  windows of gsct_voxelize_fwd tile voxelize_full bit for bit; fp64 slab moments of
  gsct_voxelize_bwd_moments all-reduced and finished equal voxelize_backward of the oracle.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_2604_01844_b200 import gsct, sharding
from conftest import grad_class_errors

pytestmark = pytest.mark.gpu

TOL = 1e-4
KEYS = ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm")


def _scene():
    cloud = gsct.make_cloud("random", 300, seed=91, pos_range=6.0)
    angles = list(np.linspace(0.0, 2 * np.pi, 9, endpoint=False))
    geom = gsct.ScanGeometry("cone", 96, 80, 0.5, 0.5, angles, 50.0, 25.0)
    gimgs = np.random.default_rng(5).uniform(-1, 1, size=(9, 80, 96)).astype(np.float32)
    grid = gsct.GridSpec.centered((40, 36, 30), 0.4)
    gvol = np.random.default_rng(6).uniform(-1, 1, size=(30, 36, 40)).astype(np.float32)
    return cloud, geom, gimgs, grid, gvol


def _np_grads(g):
    return {k: (getattr(g, k).cpu().numpy() if hasattr(getattr(g, k), "cpu") else np.asarray(getattr(g, k)))
            for k in KEYS + ("visible",)}


def test_native_group_world1_bit_identical(ctx):
    """Grouped calls at world size 1 == ungrouped calls, bitwise (the all-reduce of one rank
    is a copy; the slab of rank 0 of 1 is the whole grid)."""
    import torch

    cloud, geom, gimgs, grid, gvol = _scene()
    d = cloud.to_device(0)
    region = gsct.GridRegion.covering(grid)
    rs, vs = gsct.RasterSettings(), gsct.VoxelSettings()
    g0 = _np_grads(gsct.rasterize_backward_views(d, geom, None, torch.from_numpy(gimgs).cuda(), rs, ctx=ctx))
    v0 = gsct.voxelize(d, region, vs, ctx=ctx).cpu().numpy()
    b0 = _np_grads(gsct.voxelize_backward(d, region, torch.from_numpy(gvol).cuda(), vs, ctx=ctx))
    grp = ctx.create_group(ctx.group_new_id(), 1, 0)
    try:
        assert (grp.rank, grp.size) == (0, 1)
        g1 = _np_grads(gsct.rasterize_backward_views(d, geom, None, torch.from_numpy(gimgs).cuda(), rs, ctx=ctx))
        v1 = gsct.voxelize(d, region, vs, ctx=ctx).cpu().numpy()
        b1 = _np_grads(gsct.voxelize_backward(d, region, torch.from_numpy(gvol).cuda(), vs, ctx=ctx))
        # host buffers through the grouped path too
        g2 = gsct.rasterize_backward_views(cloud, geom, None, gimgs, rs, ctx=ctx)
    finally:
        ctx.set_group(None)
        grp.close()
    for k in KEYS + ("visible",):
        assert np.array_equal(g0[k], g1[k]), k
        assert np.array_equal(b0[k], b1[k]), k
        assert np.array_equal(g0[k], np.asarray(getattr(g2, k))), k
    assert np.array_equal(v0, v1)


def test_native_group_rejects_bad_rank(ctx):
    with pytest.raises(gsct.ContractError):
        ctx.create_group(bytes(128), 2, 2)


# ---- world size 2: the CUDA operators per rank ----------------------------------------
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = gsct.context(0)
    cloud, geom, gimgs, grid, gvol = _scene()
    n = cloud.size()
    d = cloud.to_device(0)
    rs, vs = gsct.RasterSettings(), gsct.VoxelSettings()
    # views: this rank's round-robin shard through gsct_rasterize_bwd, packed, all-reduced
    views = sharding.shard_views(len(geom.angles), rank, world)
    flat, pg = sharding.pack_grads(n, like=torch.empty(0, device="cuda"))
    gsct.rasterize_backward_views(d, geom, views, torch.from_numpy(gimgs[views]).cuda(), rs, out=pg, ctx=ctx)
    flat_c, vis_c = flat.cpu(), pg.visible.cpu()
    sharding.allreduce_grads(flat_c, vis_c)
    # voxels: this rank's z-slab of the forward; fp64 slab moments, all-reduced, finished
    region = gsct.GridRegion.covering(grid)
    (lo, hi) = sharding.zslab_windows(grid.dims, world)[rank]
    slab = gsct.voxelize(d, region, vs, window=(lo, hi), ctx=ctx).cpu()
    slabs = [None] * world
    dist.all_gather_object(slabs, (lo[2], slab.numpy()))
    mom = torch.zeros((10, n), dtype=torch.float64, device="cuda")
    gsct.voxelize_backward_moments(d, region, torch.from_numpy(gvol[lo[2]:hi[2]].copy()).cuda(), (lo, hi), mom, vs,
                                   ctx=ctx)
    mc = mom.cpu()
    sharding.allreduce_moments(mc)
    vg = gsct.voxelize_backward_finish(d, region, mc.cuda(), vs, ctx=ctx)
    if rank == 0:
        vol = np.zeros((grid.dims[2], grid.dims[1], grid.dims[0]), dtype=np.float32)
        for z0, s in slabs:
            vol[z0:z0 + s.shape[0]] = s
        np.savez(out_path, flat=flat_c.numpy(), vis=vis_c.numpy(), vol=vol,
                 **{"v_" + k: v for k, v in _np_grads(vg).items()})
    dist.destroy_process_group()


def test_world2_cuda_operators_match_oracle(ctx, orc, tmp_path):
    import torch.multiprocessing as mp

    out = tmp_path / "w2.npz"
    mp.start_processes(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    cloud, geom, gimgs, grid, gvol = _scene()
    n = cloud.size()
    rs, vs = gsct.RasterSettings(), gsct.VoxelSettings()
    acc = None
    for v in range(len(geom.angles)):
        g = orc.rasterize_backward(cloud, geom, v, gimgs[v].astype(np.float64), rs)
        acc = dict(g) if acc is None else {k: acc[k] + g[k] if k != "visible" else acc[k] | g[k] for k in g}
    flat = got["flat"]
    mine = {"positions": flat[:3 * n].reshape(n, 3), "log_scales": flat[3 * n:6 * n].reshape(n, 3),
            "rotations": flat[6 * n:10 * n].reshape(n, 4), "raw_densities": flat[10 * n:11 * n],
            "pos_grad_norm": flat[11 * n:12 * n]}
    errs = grad_class_errors(mine, acc)
    assert all(e <= TOL for e in errs.values()), errs
    assert np.array_equal(got["vis"].astype(bool), acc["visible"].astype(bool))
    # voxel forward: the two slabs tile voxelize_full of one process bit for bit
    region = gsct.GridRegion.covering(grid)
    full = gsct.voxelize(cloud.to_device(0), region, vs, ctx=ctx).cpu().numpy()
    assert np.array_equal(got["vol"], full)
    # voxel backward: all-reduced slab moments vs the oracle's full-grid voxelize_backward
    rv = orc.voxelize_backward(cloud, region, gvol.astype(np.float64), vs)
    errs = grad_class_errors({k: got["v_" + k] for k in KEYS}, rv)
    assert all(e <= TOL for e in errs.values()), errs
    assert np.array_equal(got["v_visible"].astype(bool), np.asarray(rv["visible"]).astype(bool))
