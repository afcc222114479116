"""World-size-2 gloo tests (CPU) of the multi-GPU decomposition (SURVEY.md 8(e),
paper_2604_01844_b200/sharding.py):

* view sharding: each rank sums the oracle gradients of its views, one all-reduce of the
  packed buffer (+ MAX of visibility) equals the single-process sum over all views;
* z-slab sharding: per-slab partial moments of the voxel backward, all-reduced, then the
  per-splat finish, equal the full-grid voxelize_backward of the oracle.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_01844_b200 import gsct, sharding

GRAD_KEYS = ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm")


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _scene():
    cloud = gsct.make_cloud("random", 12, seed=77, pos_range=5.0)
    geom = gsct.ScanGeometry("cone", 40, 40, 0.7, 0.7, list(np.linspace(0, 2 * np.pi, 7, endpoint=False)), 50.0, 25.0)
    grads = np.random.default_rng(3).uniform(-1, 1, size=(7, 40, 40))
    return cloud, geom, grads


def _view_worker(rank, world, port, out_path):
    from oracle.oracle import Orc

    _init(rank, world, port)
    orc = Orc()
    cloud, geom, gimgs = _scene()
    n = cloud.size()
    flat = torch.zeros(12 * n, dtype=torch.float64)
    vis = torch.zeros(n, dtype=torch.uint8)
    for v in sharding.shard_views(len(geom.angles), rank, world):
        g = orc.rasterize_backward(cloud, geom, v, gimgs[v], gsct.RasterSettings())
        flat += torch.from_numpy(np.concatenate([g["positions"].ravel(), g["log_scales"].ravel(),
                                                 g["rotations"].ravel(), g["raw_densities"], g["pos_grad_norm"]]))
        vis |= torch.from_numpy(g["visible"])
    sharding.allreduce_grads(flat, vis)
    if rank == 0:
        np.savez(out_path, flat=flat.numpy(), vis=vis.numpy())
    dist.destroy_process_group()


def test_view_sharded_gradients_equal_single_process_sum(orc, tmp_path):
    out = tmp_path / "views.npz"
    mp.spawn(_view_worker, args=(2, free_port(), str(out)), nprocs=2, join=True)
    got = np.load(out)
    cloud, geom, gimgs = _scene()
    acc = None
    vis = None
    for v in range(len(geom.angles)):
        g = orc.rasterize_backward(cloud, geom, v, gimgs[v], gsct.RasterSettings())
        flat = np.concatenate([g["positions"].ravel(), g["log_scales"].ravel(), g["rotations"].ravel(),
                               g["raw_densities"], g["pos_grad_norm"]])
        acc = flat if acc is None else acc + flat
        vis = g["visible"] if vis is None else vis | g["visible"]
    scale = np.max(np.abs(acc))
    assert np.max(np.abs(got["flat"] - acc)) <= 1e-12 * scale
    assert np.array_equal(got["vis"], vis)


def test_shard_views_and_zslabs_partition():
    for world in (1, 2, 3, 8):
        owned = sorted(v for r in range(world) for v in sharding.shard_views(75, r, world))
        assert owned == list(range(75))
        wins = sharding.zslab_windows((30, 20, 37), world)
        zs = [z for (lo, hi) in wins for z in range(lo[2], hi[2])]
        assert zs == list(range(37))
        assert all(lo[:2] == (0, 0) and hi[:2] == (30, 20) for lo, hi in wins)
    with pytest.raises(ValueError):
        sharding.shard_views(75, 2, 2)


# ---- z-slab backward: partial moments (numpy restatement of the moment definition) ----
def _activate(cloud, i):
    s = np.exp(cloud.log_scales[i])
    q = cloud.rotations[i] / np.linalg.norm(cloud.rotations[i])
    w, x, y, z = q
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    return s, q, R


def _moments(cloud, grid, gv, window, lo, hi, skip):
    """[10, N] sums over the window of t, t d, t d d^T (d in world units), t = exp(-q/2) w."""
    n = cloud.size()
    m = np.zeros((10, n))
    (x0, y0, z0), (x1, y1, z1) = window
    for i in range(n):
        if skip[i]:
            continue
        s, q, R = _activate(cloud, i)
        A = np.linalg.inv(R @ np.diag(s * s) @ R.T)
        zs = range(max(lo[i, 2], z0), min(hi[i, 2], z1 - 1) + 1)
        for zz in zs:
            for yy in range(max(lo[i, 1], y0), min(hi[i, 1], y1 - 1) + 1):
                for xx in range(max(lo[i, 0], x0), min(hi[i, 0], x1 - 1) + 1):
                    d = np.array(grid.origin) + grid.spacing * np.array([xx, yy, zz]) - cloud.positions[i]
                    t = np.exp(-0.5 * d @ A @ d) * gv[zz, yy, xx]
                    m[0, i] += t
                    m[1:4, i] += t * d
                    m[4:7, i] += t * d * d
                    m[7, i] += t * d[0] * d[1]
                    m[8, i] += t * d[0] * d[2]
                    m[9, i] += t * d[1] * d[2]
    return m


def _finish(cloud, m, skip):
    """voxelizer.hpp:250-255 + covariance_backward (core.hpp:170-191) from the moments."""
    n = cloud.size()
    out = {k: np.zeros((n, w)) if w > 1 else np.zeros(n) for k, w in
           (("positions", 3), ("log_scales", 3), ("rotations", 4), ("raw_densities", 1), ("pos_grad_norm", 1))}
    for i in range(n):
        if skip[i]:
            continue
        s, q, R = _activate(cloud, i)
        rho = max(cloud.raw_densities[i], 0.0)
        A = np.linalg.inv(R @ np.diag(s * s) @ R.T)
        gp = rho * A @ m[1:4, i]
        M2 = np.array([[m[4, i], m[7, i], m[8, i]], [m[7, i], m[5, i], m[9, i]], [m[8, i], m[9, i], m[6, i]]])
        gsig = -A @ (-0.5 * rho * M2) @ A
        Nm = R @ np.diag(s)
        gN = (gsig + gsig.T) @ Nm
        gls = s * np.diag(R.T @ gN)
        grot = gN @ np.diag(s)
        r_, x, y, z = q
        dm = [np.array([[0, -2 * z, 2 * y], [2 * z, 0, -2 * x], [-2 * y, 2 * x, 0]]),
              np.array([[0, 2 * y, 2 * z], [2 * y, -4 * x, -2 * r_], [2 * z, 2 * r_, -4 * x]]),
              np.array([[-4 * y, 2 * x, 2 * r_], [2 * x, 0, 2 * z], [-2 * r_, 2 * z, -4 * y]]),
              np.array([[-4 * z, -2 * r_, 2 * x], [2 * r_, -4 * z, 2 * y], [2 * x, 2 * y, 0]])]
        gu = np.array([np.sum(grot * d) for d in dm])
        out["positions"][i] = gp
        out["log_scales"][i] = gls
        out["rotations"][i] = (gu - q * (q @ gu)) / np.linalg.norm(cloud.rotations[i])
        out["raw_densities"][i] = m[0, i] if cloud.raw_densities[i] >= 0 else 0.0
        out["pos_grad_norm"][i] = np.linalg.norm(gp)
    return out


def _slab_worker(rank, world, port, out_path):
    from oracle.oracle import Orc

    _init(rank, world, port)
    cloud, grid, gv, vs = _voxel_scene()
    region = gsct.GridRegion.covering(grid)
    lo, hi, skip = Orc().prepare_voxel_splats(cloud, region, vs)
    win = sharding.zslab_windows(grid.dims, world)[rank]
    m = torch.from_numpy(_moments(cloud, grid, gv, win, lo, hi, skip))
    sharding.allreduce_moments(m)
    if rank == 0:
        np.save(out_path, m.numpy())
    dist.destroy_process_group()


def _voxel_scene():
    cloud = gsct.make_cloud("random", 5, seed=61, pos_range=3.0, scale_lo=0.6, scale_hi=1.4)
    grid = gsct.GridSpec.centered((12, 12, 13), 0.8)
    gv = np.random.default_rng(3).uniform(-1, 1, size=(13, 12, 12))
    return cloud, grid, gv, gsct.VoxelSettings()


def test_zslab_backward_moments_allreduce_equal_full_backward(orc, tmp_path):
    out = tmp_path / "m.npy"
    mp.spawn(_slab_worker, args=(2, free_port(), str(out)), nprocs=2, join=True)
    cloud, grid, gv, vs = _voxel_scene()
    region = gsct.GridRegion.covering(grid)
    lo, hi, skip = orc.prepare_voxel_splats(cloud, region, vs)
    got = _finish(cloud, np.load(out), skip)
    ref = orc.voxelize_backward(cloud, region, gv, vs)
    for k in GRAD_KEYS:
        scale = np.max(np.abs(ref[k]))
        assert np.max(np.abs(got[k] - ref[k])) <= 1e-9 * scale, k
