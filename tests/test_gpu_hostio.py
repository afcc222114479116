"""Pageable host buffers through the C ABI (csrc/hostio.cu): staged transfers and the
pageable host-cloud replica, the path the C++ drop-in takes (std::vector clouds, images,
gradients). Every result must be bit-identical to the device-resident call on the same
inputs, including after the caller edits the cloud in place between calls (the replica's
chunk comparison must see every change)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2604_01844_b200 import gsct

pytestmark = pytest.mark.gpu

KEYS = ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm", "visible")


def _host(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def _same_grads(a, b):
    for k in KEYS:
        assert np.array_equal(_host(getattr(a, k)), _host(getattr(b, k))), k


def test_pageable_cloud_replica_tracks_in_place_edits(ctx):
    import torch

    # 60k splats: the cloud spans many 1 MB replica chunks
    cloud = gsct.make_cloud("random", 60_000, seed=17, pos_range=8.0)
    geom = gsct.ScanGeometry("cone", 256, 256, 0.12, 0.12, [0.1, 0.9, 2.0], 50.0, 25.0)
    gimg = np.random.default_rng(2).uniform(-1, 1, size=(3, 256, 256)).astype(np.float32)
    grid = gsct.GridSpec.centered((48, 48, 48), 0.35)
    region = gsct.GridRegion.covering(grid)
    gvol = np.random.default_rng(3).uniform(-1, 1, size=(48, 48, 48)).astype(np.float32)
    for step in range(4):
        if step:  # the caller edits its arrays in place (Adam-like), same pointers
            rng = np.random.default_rng(100 + step)
            idx = rng.integers(0, cloud.size(), size=7 * step)
            cloud.positions[idx] += rng.normal(0, 0.05, size=(idx.size, 3))
            cloud.log_scales[idx[:2]] -= 0.01
            cloud.rotations[idx[-1]] = (0.5, 0.5, 0.5, 0.5)
            cloud.raw_densities[idx[0]] *= 1.5
            if step == 3:  # one change in the very last bytes of the last array
                cloud.raw_densities[-1] += 0.25
        dev = cloud.to_device(0)
        img_h = gsct.rasterize_views(cloud, geom, None, ctx=ctx)
        img_d = gsct.rasterize_views(dev, geom, None, ctx=ctx).cpu().numpy()
        assert np.array_equal(img_h, img_d), step
        g_h = gsct.rasterize_backward_views(cloud, geom, None, gimg, ctx=ctx)
        g_d = gsct.rasterize_backward_views(dev, geom, None, torch.from_numpy(gimg).cuda(), ctx=ctx)
        _same_grads(g_h, g_d)
        v_h = gsct.voxelize(cloud, region, ctx=ctx)
        v_d = gsct.voxelize(dev, region, ctx=ctx).cpu().numpy()
        assert np.array_equal(v_h, v_d), step
        b_h = gsct.voxelize_backward(cloud, region, gvol, ctx=ctx)
        b_d = gsct.voxelize_backward(dev, region, torch.from_numpy(gvol).cuda(), ctx=ctx)
        _same_grads(b_h, b_d)


def test_pageable_cloud_replica_new_arrays_and_sizes(ctx):
    """A different cloud (new pointers / size) after a cached one is uploaded in full."""
    geom = gsct.ScanGeometry("parallel", 128, 128, 0.1, 0.1, [0.3])
    for seed, n in ((1, 40_000), (2, 40_000), (3, 25_000), (1, 40_000)):
        cloud = gsct.make_cloud("random", n, seed=seed, pos_range=5.0)
        a = gsct.rasterize_views(cloud, geom, None, ctx=ctx)
        b = gsct.rasterize_views(cloud.to_device(0), geom, None, ctx=ctx).cpu().numpy()
        assert np.array_equal(a, b), (seed, n)


def test_sparse_voxel_gradients_into_zero_filled_host_buffers(ctx):
    """GSCT_HOST_ZEROED: voxelize_backward of a 32^3 sub-region (the training loop's TV term)
    brings down only the touched splats' rows; the zero-filled host output must equal the
    dense host output and the device-resident result bit for bit (every splat, visible flags
    included), also for a region no splat touches and for the full grid."""
    cloud = gsct.make_cloud("shepp_logan", 40_000, seed=3, side=128, spacing=1.0)
    grid = gsct.GridSpec.centered((128, 128, 128), 1.0)
    dcloud = cloud.to_device(0)
    rng = np.random.default_rng(5)
    for region in (gsct.GridRegion.of_parent(grid, (40, 50, 60), (32, 32, 32)),
                   gsct.GridRegion.of_parent(grid, (0, 0, 0), (4, 4, 4)),
                   gsct.GridRegion.covering(grid)):
        gv = rng.uniform(-1, 1, size=(region.dims[2], region.dims[1], region.dims[0])).astype(np.float32)
        sparse = gsct.voxelize_backward(cloud, region, gv, ctx=ctx)  # library-allocated zeros: sparse rows
        dense = gsct.voxelize_backward(cloud, region, gv, out=gsct.ParamGradients.zeros(cloud.size()), ctx=ctx)
        dev = gsct.voxelize_backward(dcloud, region, gv, ctx=ctx)
        _same_grads(sparse, dense)
        _same_grads(sparse, dev)
