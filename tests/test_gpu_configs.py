"""Parity at every BASELINE.json configuration, against the UNCHANGED reference compiled here
(oracle/_ref, all host threads), and bit-exactness of the binning the forward actually runs.

  C1 (CPU-runnable oracle config): 50k Gaussians, 128^3, 75 cone views at 256^2 --
      every view's RenderStats exact, all 75 images, the 75-view gradient sum (seeded U(-1,1)
      grad images) and voxelize_full + voxelize_backward on 128^3.
  C2 (paper standard): the 75-view all-ones gradient sum (the bench's step) vs
      sum_v rasterize_backward (ParamGradients::add, core.hpp:152-162).
  C3 (voxel fit, 512^3 / 500k): voxelize_backward on a 16-slice region vs the reference,
      directly and through the z-slab moments / finish split (voxelizer.hpp:214-263).
  C4 (1024^2 / 400k): three views, counters exact, images and gradients in tolerance.
  Forward binning (gsct_debug_fwd_bins = the forward's own 32x32 super-tile lists, packed
      narrow / wide / key+value plans) vs bin_tiles(tile_size=32) (projector.hpp:266-286):
      all 75 C2 views, one full C5 view chunk, a multi-view wide-packed case with n not a
      multiple of 4096, and n >= 2^24 splats on a small detector.
Tolerances as everywhere: images / volumes max|d| <= 1e-4 max|ref|, gradients per class
max|d| <= 1e-4 max|g_ref|; integer outputs exact.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from conftest import grad_class_errors, max_err_rel_peak
from paper_2604_01844_b200 import gsct

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _sl_workload(side, n, views, det, seed=0):
    cloud = gsct.make_cloud("shepp_logan", n, seed=seed, side=side, spacing=1.0)
    geom = gsct.default_geometry((side,) * 3, 1.0, views, "cone", det, det)
    return cloud, geom


def _ref_bins(ref, h, geom, view, n, rs32):
    """Reference bin_tiles at tile_size 32 for one view (CSR)."""
    b = ref.project_and_bin(h, geom, view, rs32, n)
    return b["tile_offsets"], b["tile_splats"]


def _check_bins(ref, cloud, geom, views, rs=gsct.RasterSettings(), ctx=None, check_views=None):
    offsets, splats = gsct.forward_bins(cloud, geom, views, rs, ctx=ctx)
    n_st = ((geom.n_u + 31) // 32) * ((geom.n_v + 31) // 32)
    rs32 = dataclasses.replace(rs, tile_size=32)
    h = ref.cloud(cloud)
    try:
        for j, v in enumerate(views):
            if check_views is not None and v not in check_views:
                continue
            ro, rsp = _ref_bins(ref, h, geom, v, cloud.size(), rs32)
            o = offsets[j * n_st:(j + 1) * n_st + 1] - offsets[j * n_st]
            assert np.array_equal(o, ro), f"view {v}: per-tile list lengths differ"
            assert np.array_equal(splats[offsets[j * n_st]:offsets[(j + 1) * n_st]].astype(np.int64),
                                  rsp.astype(np.int64)), f"view {v}: splat lists differ"
    finally:
        ref.free_cloud(h)


# --------------------------------------------------------------------------- binning
def test_forward_bins_c2_all_views(ctx, ref):
    cloud, geom = _sl_workload(256, 200_000, 75, 512)
    _check_bins(ref, cloud, geom, list(range(75)), ctx=ctx)


def test_forward_bins_c5_chunk(ctx, ref):
    """C5: the wide packed plan (tile << 20 | splat); 25 views = one forward chunk."""
    cloud, geom = _sl_workload(1024, 1_000_000, 75, 2048)
    views = list(range(25))
    _check_bins(ref, cloud, geom, views, ctx=ctx, check_views={0, 12, 24})


def test_forward_bins_and_images_wide_multiview(ctx, ref, orc):
    """> 256 super-tiles (600^2: 19 x 19), 3 views, n = 5000 (not a multiple of 4096): the
    wide packed plan with 4096-item emission CTAs spanning two views."""
    cloud = gsct.make_cloud("random", 5000, seed=3, pos_range=40.0, scale_lo=0.3, scale_hi=2.5)
    geom = gsct.ScanGeometry("cone", 600, 600, 0.15, 0.15, [0.1, 1.3, 2.9], 200.0, 100.0)
    views = [0, 1, 2]
    _check_bins(ref, cloud, geom, views, ctx=ctx)
    imgs = gsct.rasterize_views(cloud, geom, views, ctx=ctx)
    for v in views:
        single = gsct.rasterize_views(cloud, geom, [v], ctx=ctx)[0]
        assert np.array_equal(single, imgs[v])  # per-view calls: same lists, same sums
        rimg, _ = orc.rasterize_view(cloud, geom, v, gsct.RasterSettings())
        assert max_err_rel_peak(imgs[v], rimg) <= TOL


def test_forward_bins_beyond_2pow24_splats(ctx, ref):
    """n >= 2^24 on a 64^2 detector (4 super-tiles): the wide packed plan with a 30-bit
    splat field (the narrow 24-bit layout must not be used here)."""
    n = (1 << 24) + 1000
    cloud = gsct.make_cloud("random", n, seed=5, pos_range=20.0, scale_lo=0.05, scale_hi=0.3)
    geom = gsct.ScanGeometry("parallel", 64, 64, 0.7, 0.7, [0.4])
    rs = gsct.RasterSettings()
    _check_bins(ref, cloud, geom, [0], rs, ctx=ctx)
    st = gsct.RenderStats()
    img = gsct.rasterize_views(cloud, geom, [0], rs, st, ctx=ctx)[0]
    h = ref.cloud(cloud)
    try:
        rimg, rst = ref.rasterize_view(h, geom, 0, rs)
    finally:
        ref.free_cloud(h)
    assert (st.tile_pairs, st.pixel_pairs, st.culled) == (rst["tile_pairs"], rst["pixel_pairs"], rst["culled"])
    assert max_err_rel_peak(img, rimg) <= TOL


# --------------------------------------------------------------------------- C1
def test_c1_full_config(ctx, ref):
    cloud, geom = _sl_workload(128, 50_000, 75, 256)
    rs = gsct.RasterSettings()
    n = cloud.size()
    rng = np.random.default_rng(11)
    gi = rng.uniform(-1, 1, size=(75, 256, 256)).astype(np.float32)
    imgs = gsct.rasterize_views(cloud, geom, None, rs, ctx=ctx)
    g = gsct.rasterize_backward_views(cloud, geom, None, gi, rs, ctx=ctx)
    h = ref.cloud(cloud)
    try:
        acc = None
        for v in range(75):
            st = gsct.RenderStats()
            gsct.rasterize_views(cloud, geom, [v], rs, st, ctx=ctx)
            rimg, rst = ref.rasterize_view(h, geom, v, rs)
            assert (st.culled, st.degenerate, st.tile_pairs, st.pixel_pairs) == \
                (rst["culled"], rst["degenerate"], rst["tile_pairs"], rst["pixel_pairs"]), v
            assert max_err_rel_peak(imgs[v], rimg) <= TOL, v
            rg = ref.rasterize_backward(h, geom, v, gi[v].astype(np.float64), rs, n)
            if acc is None:
                acc = rg
            else:  # ParamGradients::add in ascending view order (core.hpp:152-162)
                for k in acc:
                    acc[k] = (acc[k] | rg[k]) if k == "visible" else acc[k] + rg[k]
        errs = grad_class_errors(g, acc)
        assert all(e <= TOL for e in errs.values()), errs
        assert np.array_equal(g.visible.astype(bool), acc["visible"].astype(bool))
        # voxelize_full + voxelize_backward on 128^3
        grid = gsct.GridSpec.centered((128,) * 3, 1.0)
        region = gsct.GridRegion.covering(grid)
        vs = gsct.VoxelSettings()
        st = gsct.RenderStats()
        vol = gsct.voxelize(cloud, region, vs, st, ctx=ctx)
        rvol, rst = ref.voxelize(h, region, vs)
        assert (st.culled, st.pixel_pairs) == (rst["culled"], rst["pixel_pairs"])
        assert max_err_rel_peak(vol, rvol) <= TOL
        gv = rng.uniform(-1, 1, size=vol.shape).astype(np.float32)
        vg = gsct.voxelize_backward(cloud, region, gv, vs, ctx=ctx)
        rvg = ref.voxelize_backward(h, region, gv.astype(np.float64), vs, n)
    finally:
        ref.free_cloud(h)
    errs = grad_class_errors(vg, rvg)
    assert all(e <= TOL for e in errs.values()), errs


# --------------------------------------------------------------------------- C2
def test_c2_all_views_gradient_sum(ctx, ref):
    """The bench's step: 75 views, all-ones grad images (bench.hpp:114-115), gradients summed
    over views, against sum_v Ref.rasterize_backward."""
    cloud, geom = _sl_workload(256, 200_000, 75, 512)
    rs = gsct.RasterSettings()
    n = cloud.size()
    g = gsct.rasterize_backward_views(cloud, geom, None, np.ones((75, 512, 512), np.float32), rs, ctx=ctx)
    ones = np.ones((512, 512))
    h = ref.cloud(cloud)
    try:
        acc = None
        for v in range(75):
            rg = ref.rasterize_backward(h, geom, v, ones, rs, n)
            if acc is None:
                acc = rg
            else:
                for k in acc:
                    acc[k] = (acc[k] | rg[k]) if k == "visible" else acc[k] + rg[k]
    finally:
        ref.free_cloud(h)
    errs = grad_class_errors(g, acc)
    assert all(e <= TOL for e in errs.values()), errs
    assert np.array_equal(g.visible.astype(bool), acc["visible"].astype(bool))


# --------------------------------------------------------------------------- C3
def test_c3_voxel_backward_slab(ctx, ref):
    import torch

    side, n = 512, 500_000
    cloud = gsct.make_cloud("shepp_logan", n, seed=1, side=side, spacing=1.0)
    grid = gsct.GridSpec.centered((side,) * 3, 1.0)
    vs = gsct.VoxelSettings()
    z0, dz = 248, 16
    region = gsct.GridRegion.of_parent(grid, (0, 0, z0), (side, side, dz))
    gv = np.random.default_rng(21).uniform(-1, 1, size=(dz, side, side)).astype(np.float32)
    g = gsct.voxelize_backward(cloud, region, gv, vs, ctx=ctx)
    h = ref.cloud(cloud)
    try:
        rg = ref.voxelize_backward(h, region, gv.astype(np.float64), vs, n)
    finally:
        ref.free_cloud(h)
    errs = grad_class_errors(g, rg)
    assert all(e <= TOL for e in errs.values()), errs
    assert np.array_equal(g.visible.astype(bool), rg["visible"].astype(bool))
    # the z-slab sharded path: moments over the window of the full grid, then the finish
    d = cloud.to_device(0)
    full = gsct.GridRegion.covering(grid)
    mom = torch.zeros((10, n), dtype=torch.float64, device="cuda")
    gsct.voxelize_backward_moments(d, full, torch.from_numpy(gv).cuda(), ((0, 0, z0), (side, side, z0 + dz)), mom,
                                   vs, ctx=ctx)
    gm = gsct.voxelize_backward_finish(d, full, mom, vs, ctx=ctx)
    gm = {k: getattr(gm, k).cpu().numpy() for k in ("positions", "log_scales", "rotations", "raw_densities",
                                                     "pos_grad_norm", "visible")}
    errs = grad_class_errors(gm, rg)
    assert all(e <= TOL for e in errs.values()), errs


# --------------------------------------------------------------------------- C4
def test_c4_three_views(ctx, ref):
    cloud, geom = _sl_workload(512, 400_000, 75, 1024)
    rs = gsct.RasterSettings()
    h = ref.cloud(cloud)
    try:
        for v in (0, 25, 50):
            st = gsct.RenderStats()
            img = gsct.rasterize_views(cloud, geom, [v], rs, st, ctx=ctx)[0]
            rimg, rst = ref.rasterize_view(h, geom, v, rs)
            assert (st.culled, st.degenerate, st.tile_pairs, st.pixel_pairs) == \
                (rst["culled"], rst["degenerate"], rst["tile_pairs"], rst["pixel_pairs"]), v
            assert max_err_rel_peak(img, rimg) <= TOL, v
            gi = np.random.default_rng(40 + v).uniform(-1, 1, size=img.shape).astype(np.float32)
            g = gsct.rasterize_backward_views(cloud, geom, [v], gi[None], rs, ctx=ctx)
            rg = ref.rasterize_backward(h, geom, v, gi.astype(np.float64), rs, cloud.size())
            errs = grad_class_errors(g, rg)
            assert all(e <= TOL for e in errs.values()), (v, errs)
    finally:
        ref.free_cloud(h)


@pytest.mark.parametrize("det,n,bounding,dilate", [(600, 5000, "square_circumscribed", False),
                                                   (256, 20000, "rect_density_aware", True)])
def test_parallel_beam_bins_images_gradients(ctx, ref, orc, det, n, bounding, dilate):
    """Parallel-beam geometry through the packed binning the forward ships (wide layout at
    600^2 with > 256 super-tiles, narrow at 256^2, n >= 4096), with square bounding /
    no dilation: lists bit-exact vs bin_tiles, images and gradients vs the oracle."""
    cloud = gsct.make_cloud("random", n, seed=9, pos_range=30.0, scale_lo=0.3, scale_hi=2.0)
    geom = gsct.ScanGeometry("parallel", det, det, 0.12, 0.12, [0.2, 1.7, 4.1], 0.0, 0.0)
    rs = gsct.RasterSettings(bounding=bounding, dilate=dilate)
    views = [0, 1, 2]
    _check_bins(ref, cloud, geom, views, rs=rs, ctx=ctx)
    imgs = gsct.rasterize_views(cloud, geom, views, rs, ctx=ctx)
    gi = np.random.default_rng(4).uniform(-1, 1, size=imgs.shape).astype(np.float32)
    g = gsct.rasterize_backward_views(cloud, geom, [1], gi[1:2], rs, ctx=ctx)
    for v in views:
        rimg, _ = orc.rasterize_view(cloud, geom, v, rs)
        assert max_err_rel_peak(imgs[v], rimg) <= TOL
    r = orc.rasterize_backward(cloud, geom, 1, gi[1].astype(np.float64), rs)
    errs = grad_class_errors(g, r)
    assert all(e <= TOL for e in errs.values()), errs
