"""GPU parity of the rasterizer (C ABI via paper_2604_01844_b200.gsct) against the CPU oracle.

Gates (BASELINE north_star):
  * bounding boxes, culled/degenerate flags, tile lists, RenderStats counters: bit-exact
    (a mismatch is only tolerated as a reported "tie" when the oracle's m +- h lies within
    1e-9 of an integer, i.e. a 1-ulp libdevice-vs-glibc transcendental difference);
  * images: max|d| <= 1e-4 * max|ref| (fp32 per-pair math vs the fp64 oracle);
  * gradients: per parameter class max|d| <= 1e-4 * max|g_ref|;
  * determinism: bit-identical results run to run; duplicated splats get identical grads."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import (cone_geometry, grad_class_errors, max_err_rel_peak, oracle_settings,
                      parallel_geometry)
from paper_2604_01844_b200 import gsct

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4
GRAD_TOL = 1e-4

GEOMS = {
    "parallel": lambda: parallel_geometry(52, 0.55, [0.3, 2.4, 5.0]),
    "cone": lambda: cone_geometry(48, 0.7, [0.9, 2.5, 4.1]),
}
SETTINGS = {"default": gsct.RasterSettings(), "oracle": oracle_settings()}


def _ties(orc_pc, dev_pc, cloud, geom, view, rs) -> np.ndarray:
    """Indices where rects differ; each must be a near-integer tie."""
    bad = np.nonzero(np.any(orc_pc["rect"] != dev_pc["rect"], axis=1) | (orc_pc["culled"] != dev_pc["culled"]))[0]
    return bad


@pytest.mark.parametrize("gname", list(GEOMS))
@pytest.mark.parametrize("sname", list(SETTINGS))
def test_project_and_bin_bit_exact(ctx, orc, gname, sname):
    geom = GEOMS[gname]()
    rs = SETTINGS[sname]
    cloud = gsct.make_cloud("random", 200, seed=35, pos_range=8.0)
    for view in range(len(geom.angles)):
        op = orc.project_cloud(cloud, geom, view, rs)
        dp = gsct.project_cloud(cloud, geom, view, rs, ctx=ctx)
        assert np.array_equal(op["degenerate"], dp["degenerate"])
        bad = _ties(op, dp, cloud, geom, view, rs)
        assert bad.size == 0, f"bbox mismatch at splats {bad[:10]}"
        vis = ~(op["culled"] | op["degenerate"])
        # fp64 splat set-up follows the reference operation order: values agree to ~ulps
        np.testing.assert_allclose(dp["mean2d"][vis], op["mean2d"][vis], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(dp["conic"][vis], op["conic"][vis], rtol=1e-11, atol=1e-14)
        np.testing.assert_allclose(dp["amplitude"][vis], op["amplitude"][vis], rtol=1e-11)
        # tile lists (key = tile, value = splat; ascending splat index within a tile)
        off, vals = orc.bin_tiles(cloud, geom, view, rs)
        keys, dvals = gsct.tile_pairs(cloud, geom, [view], rs, ctx=ctx)
        ts = rs.tile_size
        n_tiles = ((geom.n_u + ts - 1) // ts) * ((geom.n_v + ts - 1) // ts)
        okeys = np.repeat(np.arange(n_tiles, dtype=np.uint32), np.diff(off))
        assert np.array_equal(keys, okeys)
        assert np.array_equal(dvals.astype(np.int32), vals)


def test_multiview_keys_bit_exact(ctx, orc):
    geom = cone_geometry(64, 0.5, np.linspace(0, 2 * np.pi, 9, endpoint=False))
    rs = gsct.RasterSettings()
    cloud = gsct.make_cloud("random", 300, seed=3, pos_range=9.0, scale_lo=0.3, scale_hi=1.5)
    keys, vals = gsct.tile_pairs(cloud, geom, None, rs, ctx=ctx)
    n_tiles = 16
    ok, ov = [], []
    for view in range(len(geom.angles)):
        off, v = orc.bin_tiles(cloud, geom, view, rs)
        ok.append(view * n_tiles + np.repeat(np.arange(n_tiles), np.diff(off)))
        ov.append(v)
    assert np.array_equal(keys, np.concatenate(ok).astype(np.uint32))
    assert np.array_equal(vals.astype(np.int32), np.concatenate(ov))


@pytest.mark.parametrize("gname", list(GEOMS))
@pytest.mark.parametrize("sname", list(SETTINGS))
def test_forward_matches_oracle(ctx, orc, gname, sname):
    geom = GEOMS[gname]()
    rs = SETTINGS[sname]
    cloud = gsct.make_cloud("random", 60, seed=34)
    stats = gsct.RenderStats()
    imgs = gsct.rasterize_views(cloud, geom, None, rs, stats, ctx=ctx)
    tot = dict(culled=0, degenerate=0, tile_pairs=0, pixel_pairs=0)
    for view in range(len(geom.angles)):
        ref_img, st = orc.rasterize_view(cloud, geom, view, rs)
        assert max_err_rel_peak(imgs[view], ref_img) <= IMG_TOL
        for k in tot:
            tot[k] += st[k]
    assert (stats.culled, stats.degenerate, stats.tile_pairs, stats.pixel_pairs) == (
        tot["culled"], tot["degenerate"], tot["tile_pairs"], tot["pixel_pairs"])
    assert stats.forward_ms > 0.0


@pytest.mark.parametrize("gname", list(GEOMS))
@pytest.mark.parametrize("sname", list(SETTINGS))
def test_backward_matches_oracle(ctx, orc, gname, sname):
    geom = GEOMS[gname]()
    rs = SETTINGS[sname]
    cloud = gsct.make_cloud("random", 40, seed=41 if gname == "parallel" else 42)
    cloud.raw_densities[2] = -0.3  # clamped density: gradient gated by raw >= 0
    rng = np.random.default_rng(99)
    gi = rng.uniform(-1, 1, size=(len(geom.angles), geom.n_v, geom.n_u)).astype(np.float32)
    grads = gsct.rasterize_backward_views(cloud, geom, None, gi, rs, ctx=ctx)
    # oracle: sum over views in ascending order (ParamGradients::add)
    acc = None
    for view in range(len(geom.angles)):
        g = orc.rasterize_backward(cloud, geom, view, gi[view].astype(np.float64), rs)
        if acc is None:
            acc = g
        else:
            for k in ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm"):
                acc[k] = acc[k] + g[k]
            acc["visible"] = acc["visible"] | g["visible"]
    errs = grad_class_errors(grads, acc)
    assert all(e <= GRAD_TOL for e in errs.values()), errs
    assert np.array_equal(grads.visible, acc["visible"])


def test_single_view_api_and_zero_gradient(ctx, orc):
    geom = parallel_geometry(32, 0.7, [0.5])
    cloud = gsct.make_cloud("random", 5, seed=36)
    img = gsct.rasterize_view(cloud, geom, 0, ctx=ctx)
    ref_img, _ = orc.rasterize_view(cloud, geom, 0, gsct.RasterSettings())
    assert img.shape == (32, 32) and max_err_rel_peak(img, ref_img) <= IMG_TOL
    g = gsct.rasterize_backward(cloud, geom, 0, np.zeros((32, 32), np.float32), ctx=ctx)
    for k in ("positions", "log_scales", "rotations", "raw_densities"):
        assert np.all(getattr(g, k) == 0.0)


def test_empty_cloud_and_no_views(ctx):
    geom = parallel_geometry(33, 1.0, [0.0])
    img = gsct.rasterize_view(gsct.GaussianCloud.empty(), geom, 0, ctx=ctx)
    assert np.all(img == 0.0)
    g = gsct.rasterize_backward(gsct.GaussianCloud.empty(), geom, 0, np.ones((33, 33), np.float32), ctx=ctx)
    assert g.positions.shape == (0, 3)


def test_single_splat_peak_and_exact_doubling(ctx):
    """test_projector.cpp:177-203"""
    geom = parallel_geometry(33, 1.0, [0.0])
    s = 8.0
    one = gsct.GaussianCloud(np.zeros((1, 3)), np.full((1, 3), np.log(s)), np.array([[1.0, 0, 0, 0]]),
                             np.array([0.7]))
    img = gsct.rasterize_view(one, geom, 0, ctx=ctx)
    assert img[16, 16] == pytest.approx(0.7 * np.sqrt(2 * np.pi) * s, rel=0.01)
    a = gsct.GaussianCloud(np.array([[0.5, -1, 2]]), np.full((1, 3), np.log(3.0)), np.array([[1.0, 0, 0, 0]]),
                           np.array([0.9]))
    b = gsct.GaussianCloud(np.repeat(a.positions, 2, 0), np.repeat(a.log_scales, 2, 0),
                           np.repeat(a.rotations, 2, 0), np.repeat(a.raw_densities, 2, 0))
    ia = gsct.rasterize_view(a, geom, 0, ctx=ctx)
    ib = gsct.rasterize_view(b, geom, 0, ctx=ctx)
    assert np.array_equal(ib, 2.0 * ia)


def test_density_homogeneity_power_of_two_exact(ctx):
    """test_projector.cpp:221-249: power-of-two density factors scale images exactly."""
    cloud = gsct.make_cloud("random", 6, seed=33)
    geom = parallel_geometry(40, 0.6, [0.2])
    rs = gsct.RasterSettings(tau_cut=1e-12)
    base = gsct.rasterize_view(cloud, geom, 0, rs, ctx=ctx)
    for c in (0.0, 0.5, 2.0, 4.0):
        sc = gsct.GaussianCloud(cloud.positions, cloud.log_scales, cloud.rotations, cloud.raw_densities * c)
        img = gsct.rasterize_view(sc, geom, 0, rs, ctx=ctx)
        assert np.array_equal(img, np.float32(c) * base)
    sc = gsct.GaussianCloud(cloud.positions, cloud.log_scales, cloud.rotations, cloud.raw_densities * 1.7)
    assert max_err_rel_peak(gsct.rasterize_view(sc, geom, 0, rs, ctx=ctx), 1.7 * base.astype(np.float64)) < 1e-6


def test_linearity_and_order(ctx):
    """test_projector.cpp:205-268"""
    a = gsct.make_cloud("random", 6, seed=31)
    b = gsct.make_cloud("random", 5, seed=32)
    both = gsct.GaussianCloud(*(np.concatenate([x, y]) for x, y in zip(
        (a.positions, a.log_scales, a.rotations, a.raw_densities),
        (b.positions, b.log_scales, b.rotations, b.raw_densities))))
    geom = parallel_geometry(40, 0.6, [0.8])
    ia, ib, iab = (gsct.rasterize_view(c, geom, 0, ctx=ctx).astype(np.float64) for c in (a, b, both))
    assert max_err_rel_peak(iab, ia + ib) < 1e-5
    cloud = gsct.make_cloud("random", 12, seed=34)
    base = gsct.rasterize_view(cloud, geom, 0, ctx=ctx)
    perm = gsct.GaussianCloud(cloud.positions[::-1].copy(), cloud.log_scales[::-1].copy(),
                              cloud.rotations[::-1].copy(), cloud.raw_densities[::-1].copy())
    assert max_err_rel_peak(gsct.rasterize_view(perm, geom, 0, ctx=ctx), base) < 1e-5
    for _ in range(3):
        assert np.array_equal(gsct.rasterize_view(cloud, geom, 0, ctx=ctx), base)


def test_backward_determinism_and_duplicates(ctx):
    """test_projector.cpp:366-379: duplicated splats receive identical gradients."""
    cloud = gsct.make_cloud("random", 3, seed=43)
    dup = gsct.GaussianCloud(np.concatenate([cloud.positions, cloud.positions[1:2]]),
                             np.concatenate([cloud.log_scales, cloud.log_scales[1:2]]),
                             np.concatenate([cloud.rotations, cloud.rotations[1:2]]),
                             np.concatenate([cloud.raw_densities, cloud.raw_densities[1:2]]))
    geom = parallel_geometry(32, 0.7, [0.4])
    gi = np.random.default_rng(5).uniform(-1, 1, size=(32, 32)).astype(np.float32)
    g = gsct.rasterize_backward(dup, geom, 0, gi, ctx=ctx)
    for k in ("positions", "log_scales", "rotations", "raw_densities"):
        arr = getattr(g, k)
        assert np.array_equal(arr[1], arr[3]), k
    g2 = gsct.rasterize_backward(dup, geom, 0, gi, ctx=ctx)
    for k in ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm"):
        assert np.array_equal(getattr(g, k), getattr(g2, k))


def test_degenerate_counted(ctx):
    """test_projector.cpp:381-394"""
    cloud = gsct.GaussianCloud(np.zeros((1, 3)), np.array([[np.log(1e3), np.log(1e-9), np.log(1e3)]]),
                               np.array([[1.0, 0, 0, 0]]), np.array([1.0]))
    geom = parallel_geometry(16, 1.0, [0.0])
    st = gsct.RenderStats()
    img = gsct.rasterize_view(cloud, geom, 0, gsct.RasterSettings(dilate=False), st, ctx=ctx)
    assert st.degenerate == 1
    assert np.all(img == 0.0)


def test_contract_errors(ctx):
    cloud = gsct.make_cloud("random", 10, seed=1)
    geom = parallel_geometry(16, 1.0, [0.0])
    bad = gsct.GaussianCloud(cloud.positions.copy(), cloud.log_scales, cloud.rotations, cloud.raw_densities)
    bad.positions[7, 1] = np.nan
    bad.positions[9, 0] = np.inf
    with pytest.raises(gsct.ContractError, match="non-finite parameter in splat 7"):
        gsct.rasterize_view(bad, geom, 0, ctx=ctx)
    zq = gsct.GaussianCloud(cloud.positions, cloud.log_scales, cloud.rotations.copy(), cloud.raw_densities)
    zq.rotations[4] = 0.0
    with pytest.raises(gsct.ContractError, match="zero quaternion in splat 4"):
        gsct.rasterize_backward(zq, geom, 0, np.ones((16, 16), np.float32), ctx=ctx)
    with pytest.raises(gsct.ContractError, match="detector"):
        gsct.rasterize_view(cloud, parallel_geometry(0, 1.0, [0.0]), 0, ctx=ctx)
    with pytest.raises(gsct.ContractError, match="cone distances"):
        gsct.rasterize_view(cloud, gsct.ScanGeometry("cone", 8, 8, 1, 1, [0.0]), 0, ctx=ctx)
    with pytest.raises(gsct.ContractError, match="grad image dims"):
        gsct.rasterize_backward(cloud, geom, 0, np.ones((8, 16), np.float32), ctx=ctx)
    # the context stays usable after errors
    assert np.isfinite(gsct.rasterize_view(cloud, geom, 0, ctx=ctx)).all()


def test_device_resident_matches_host(ctx):
    import torch

    geom = cone_geometry(64, 0.5, [0.1, 1.2, 3.3, 5.5])
    cloud = gsct.make_cloud("random", 150, seed=8, pos_range=8.0)
    host = gsct.rasterize_views(cloud, geom, None, ctx=ctx)
    dcloud = cloud.to_device(0)
    dev = gsct.rasterize_views(dcloud, geom, None, ctx=ctx)
    assert np.array_equal(dev.cpu().numpy(), host)
    gi = np.random.default_rng(2).uniform(-1, 1, size=host.shape).astype(np.float32)
    gh = gsct.rasterize_backward_views(cloud, geom, None, gi, ctx=ctx)
    gd = gsct.rasterize_backward_views(dcloud, geom, None, torch.from_numpy(gi).cuda(), ctx=ctx)
    for k in ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm", "visible"):
        assert np.array_equal(getattr(gd, k).cpu().numpy(), getattr(gh, k)), k


@pytest.mark.parametrize("n", [300, 5000, 20000])
def test_pinned_host_buffers_zero_copy(ctx, n):
    """Pinned (device-mapped) host images are written by the forward kernel directly
    (zero-copy); host gradients of >= 4096 splats come down in splat-range pieces behind the
    tail; a host cloud of >= 16384 splats goes up in pieces, each piece's set-up starting
    behind its bytes. Results are bit-identical to the device-resident and pageable paths, with and
    without save-for-backward."""
    import torch

    geom = cone_geometry(64, 0.5, np.linspace(0, 2 * np.pi, 7, endpoint=False))
    cloud = gsct.make_cloud("random", n, seed=12, pos_range=8.0)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    pcloud = gsct.GaussianCloud(pin(cloud.positions), pin(cloud.log_scales), pin(cloud.rotations),
                                pin(cloud.raw_densities))
    dev = gsct.rasterize_views(cloud.to_device(0), geom, None, ctx=ctx).cpu().numpy()
    img = torch.full((7, 64, 64), np.nan, dtype=torch.float32).pin_memory().numpy()
    gsct.rasterize_views(pcloud, geom, None, out=img, ctx=ctx)
    assert np.array_equal(img, dev)
    gi = pin(np.random.default_rng(5).uniform(-1, 1, size=img.shape).astype(np.float32))
    pageable = gsct.rasterize_backward_views(cloud, geom, None, np.array(gi), ctx=ctx)
    dgrad = gsct.rasterize_backward_views(cloud.to_device(0), geom, None, torch.from_numpy(np.array(gi)).cuda(),
                                          ctx=ctx)
    for k in ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm", "visible"):
        assert np.array_equal(getattr(dgrad, k).cpu().numpy(), getattr(pageable, k)), k
    z = lambda *s: torch.full(s, np.nan, dtype=torch.float64).pin_memory().numpy()
    for sfb in (False, True):
        gh = gsct.ParamGradients(z(n, 3), z(n, 3), z(n, 4), z(n), z(n),
                                 torch.full((n,), 7, dtype=torch.uint8).pin_memory().numpy())
        try:
            ctx.set_save_for_backward(sfb)
            gsct.rasterize_views(pcloud, geom, None, out=img, ctx=ctx)
            gsct.rasterize_backward_views(pcloud, geom, None, gi, out=gh, ctx=ctx)
        finally:
            ctx.set_save_for_backward(False)
        for k in ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm", "visible"):
            assert np.array_equal(getattr(gh, k), getattr(pageable, k)), (sfb, k)


def test_save_for_backward_is_exact(ctx):
    """Reusing the forward's set-up gives bit-identical gradients; a call that does not match
    the saved forward (other views) recomputes."""
    import torch

    geom = cone_geometry(64, 0.5, np.linspace(0, 2 * np.pi, 9, endpoint=False))
    cloud = gsct.make_cloud("random", 120, seed=9, pos_range=8.0).to_device(0)
    gi = torch.from_numpy(np.random.default_rng(4).uniform(-1, 1, size=(9, 64, 64)).astype(np.float32)).cuda()
    base = gsct.rasterize_backward_views(cloud, geom, None, gi, ctx=ctx)
    try:
        ctx.set_save_for_backward(True)
        gsct.rasterize_views(cloud, geom, None, ctx=ctx)
        reused = gsct.rasterize_backward_views(cloud, geom, None, gi, ctx=ctx)
        other = gsct.rasterize_backward_views(cloud, geom, [0, 1, 2], gi[:3], ctx=ctx)  # no saved match
    finally:
        ctx.set_save_for_backward(False)
    ref3 = gsct.rasterize_backward_views(cloud, geom, [0, 1, 2], gi[:3], ctx=ctx)
    for k in ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm", "visible"):
        assert torch.equal(getattr(reused, k), getattr(base, k)), k
        assert torch.equal(getattr(other, k), getattr(ref3, k)), k


def test_view_chunking_invariance(ctx, orc):
    """Many views (chunked internally) give the same per-view images as single calls."""
    geom = cone_geometry(32, 0.9, np.linspace(0, 2 * np.pi, 23, endpoint=False))
    cloud = gsct.make_cloud("random", 80, seed=77, pos_range=6.0)
    imgs = gsct.rasterize_views(cloud, geom, None, ctx=ctx)
    for v in (0, 7, 22):
        assert np.array_equal(imgs[v], gsct.rasterize_view(cloud, geom, v, ctx=ctx))


@pytest.mark.parametrize("spacing", [0.35, 0.12, 0.045])
def test_backward_bbox_size_sweep(ctx, orc, spacing):
    """Backward column-block plan across bbox regimes: W, H from a few pixels to > 128
    (the plan table's clamp / fallback paths), anisotropic splats (W != H)."""
    geom = parallel_geometry(300, spacing, [0.4, 1.9])
    rs = gsct.RasterSettings()
    cloud = gsct.make_cloud("random", 24, seed=123, pos_range=3.0, scale_lo=0.05, scale_hi=1.6)
    rng = np.random.default_rng(5)
    gi = rng.uniform(-1, 1, size=(len(geom.angles), geom.n_v, geom.n_u)).astype(np.float32)
    grads = gsct.rasterize_backward_views(cloud, geom, None, gi, rs, ctx=ctx)
    acc = None
    for view in range(len(geom.angles)):
        g = orc.rasterize_backward(cloud, geom, view, gi[view].astype(np.float64), rs)
        acc = g if acc is None else {k: (acc[k] | g[k]) if k == "visible" else acc[k] + g[k] for k in g}
    errs = grad_class_errors(grads, acc)
    assert all(e <= GRAD_TOL for e in errs.values()), errs
    pc = orc.project_cloud(cloud, geom, 0, rs)
    w = pc["rect"][:, 1] - pc["rect"][:, 0] + 1
    assert w.max() > 8  # the sweep really covers multi-block boxes


@pytest.mark.parametrize("gname", list(GEOMS))
def test_forward_extreme_shapes(ctx, orc, gname):
    """Needle-like rotated splats (whose bbox corners underflow exp in fp32: the forward's
    multiplicative row chain must fall back to the direct path) and sub-pixel splats, mixed
    with ordinary ones; forward and backward within tolerance of the oracle."""
    geom = GEOMS[gname]()
    rs = gsct.RasterSettings()
    base = gsct.make_cloud("random", 30, seed=71, pos_range=6.0)
    rng = np.random.default_rng(3)
    ls = base.log_scales.copy()
    ls[:10] = np.stack([np.full(10, -3.5), np.full(10, 1.2), np.full(10, -3.0)], axis=1)  # needles
    ls[10:20] = rng.uniform(-4.0, -2.5, size=(10, 3))                                     # sub-pixel
    cloud = gsct.GaussianCloud(base.positions, ls, base.rotations, base.raw_densities)
    imgs = gsct.rasterize_views(cloud, geom, None, rs, ctx=ctx)
    for v in range(len(geom.angles)):
        ref, _ = orc.rasterize_view(cloud, geom, v, rs)
        assert max_err_rel_peak(imgs[v], ref) <= IMG_TOL
    gi = rng.uniform(-1, 1, size=imgs.shape).astype(np.float32)
    grads = gsct.rasterize_backward_views(cloud, geom, None, gi, rs, ctx=ctx)
    acc = None
    for v in range(len(geom.angles)):
        g = orc.rasterize_backward(cloud, geom, v, gi[v].astype(np.float64), rs)
        acc = g if acc is None else {k: (acc[k] | g[k]) if k == "visible" else acc[k] + g[k] for k in g}
    errs = grad_class_errors(grads, acc)
    assert all(e <= GRAD_TOL for e in errs.values()), errs


def test_pinned_ragged_detector(ctx):
    """Zero-copy host images on a detector whose width is not a multiple of 4 (scalar-store
    edge path) and whose height is not a multiple of 16: identical to the device path."""
    import torch

    geom = gsct.ScanGeometry("cone", 50, 37, 0.6, 0.6, [0.2, 1.9, 4.4], 50.0, 25.0)
    cloud = gsct.make_cloud("random", 400, seed=21, pos_range=7.0)
    dev = gsct.rasterize_views(cloud.to_device(0), geom, None, ctx=ctx).cpu().numpy()
    img = torch.full((3, 37, 50), np.nan, dtype=torch.float32).pin_memory().numpy()
    gsct.rasterize_views(cloud, geom, None, out=img, ctx=ctx)
    assert np.array_equal(img, dev)


@pytest.mark.parametrize("sfb", [False, True])
def test_chunked_host_grads_match_device(ctx, sfb):
    """>= 12 views with host grad images: growing upload chunks, each walked as it lands
    (with save-for-backward: one all-view sort, chunk walks on two streams, tail pieces on
    two streams). Gradients bit-identical to the device-resident call."""
    import torch

    geom = cone_geometry(48, 0.6, np.linspace(0, 2 * np.pi, 23, endpoint=False))
    cloud = gsct.make_cloud("random", 6000, seed=31, pos_range=7.0)
    gi = np.random.default_rng(9).uniform(-1, 1, size=(23, 48, 48)).astype(np.float32)
    dcloud = cloud.to_device(0)
    want = gsct.rasterize_backward_views(dcloud, geom, None, torch.from_numpy(gi).cuda(), ctx=ctx)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    pcloud = gsct.GaussianCloud(pin(cloud.positions), pin(cloud.log_scales), pin(cloud.rotations),
                                pin(cloud.raw_densities))
    n = cloud.size()
    z = lambda *s: torch.full(s, np.nan, dtype=torch.float64).pin_memory().numpy()
    gh = gsct.ParamGradients(z(n, 3), z(n, 3), z(n, 4), z(n), z(n), torch.full((n,), 7, dtype=torch.uint8).pin_memory().numpy())
    img = torch.empty((23, 48, 48), dtype=torch.float32).pin_memory().numpy()
    try:
        ctx.set_save_for_backward(sfb)
        gsct.rasterize_views(pcloud, geom, None, out=img, ctx=ctx)
        gsct.rasterize_backward_views(pcloud, geom, None, pin(gi), out=gh, ctx=ctx)
    finally:
        ctx.set_save_for_backward(False)
    for k in ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm", "visible"):
        assert np.array_equal(getattr(gh, k), getattr(want, k).cpu().numpy()), (sfb, k)
