"""GPU parity of the voxelizer against the CPU oracle (boxes bit-exact; volumes within
1e-4 of peak; gradients within 1e-4 of the per-class max; z-slab windows tile the
full-grid result bit for bit)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import grad_class_errors, max_err_rel_peak
from paper_2604_01844_b200 import gsct

pytestmark = pytest.mark.gpu

VOL_TOL = 1e-4
GRAD_TOL = 1e-4

CASES = {
    "default": (gsct.GridSpec.centered((24, 26, 22), 0.7), gsct.VoxelSettings()),
    "wide": (gsct.GridSpec.centered((20, 20, 20), 0.8), gsct.VoxelSettings(tau_cut=1e-12, sigma_cap=8.0)),
    "fine": (gsct.GridSpec.centered((40, 36, 33), 0.3), gsct.VoxelSettings()),
}


@pytest.mark.parametrize("case", list(CASES))
def test_boxes_bit_exact(ctx, orc, case):
    grid, vs = CASES[case]
    cloud = gsct.make_cloud("random", 300, seed=51, pos_range=9.0, scale_lo=0.2, scale_hi=2.0)
    for region in (gsct.GridRegion.covering(grid), gsct.GridRegion.of_parent(grid, (3, 4, 5), (9, 11, 7))):
        olo, ohi, oskip = orc.prepare_voxel_splats(cloud, region, vs)
        dlo, dhi, dskip = gsct.voxel_boxes(cloud, region, vs, ctx=ctx)
        assert np.array_equal(oskip, dskip)
        assert np.array_equal(olo[~oskip], dlo[~dskip])
        assert np.array_equal(ohi[~oskip], dhi[~dskip])


@pytest.mark.parametrize("case", list(CASES))
def test_forward_matches_oracle(ctx, orc, case):
    grid, vs = CASES[case]
    cloud = gsct.make_cloud("random", 40, seed=52, pos_range=6.0)
    for region in (gsct.GridRegion.covering(grid), gsct.GridRegion.of_parent(grid, (5, 8, 2), (10, 9, 14))):
        st = gsct.RenderStats()
        vol = gsct.voxelize(cloud, region, vs, st, ctx=ctx)
        ref, rst = orc.voxelize(cloud, region, vs)
        assert vol.shape == ref.shape
        assert max_err_rel_peak(vol, ref) <= VOL_TOL
        assert st.culled == rst["culled"] and st.pixel_pairs == rst["pixel_pairs"]


@pytest.mark.parametrize("case", list(CASES))
def test_backward_matches_oracle(ctx, orc, case):
    grid, vs = CASES[case]
    cloud = gsct.make_cloud("random", 30, seed=54, pos_range=4.0)
    cloud.raw_densities[1] = -0.1
    region = gsct.GridRegion.covering(grid)
    gv = np.random.default_rng(7).uniform(-1, 1, size=(grid.dims[2], grid.dims[1], grid.dims[0]))
    g = gsct.voxelize_backward(cloud, region, gv.astype(np.float32), vs, ctx=ctx)
    r = orc.voxelize_backward(cloud, region, gv.astype(np.float32).astype(np.float64), vs)
    errs = grad_class_errors(g, r)
    assert all(e <= GRAD_TOL for e in errs.values()), errs
    assert np.array_equal(g.visible, r["visible"])


def test_peak_is_density(ctx):
    """test_voxelizer.cpp:16-22 (fp32 volume: peak == float32(rho) exactly)."""
    grid = gsct.GridSpec.centered((9, 9, 9), 1.0)
    cloud = gsct.GaussianCloud(np.zeros((1, 3)), np.full((1, 3), np.log(1.5)), np.array([[1.0, 0, 0, 0]]),
                               np.array([0.8]))
    vol = gsct.voxelize_full(cloud, grid, ctx=ctx)
    assert vol[4, 4, 4] == np.float32(0.8)


def test_empty_and_zero_grad(ctx):
    grid = gsct.GridSpec.centered((8, 8, 8), 1.0)
    vol = gsct.voxelize_full(gsct.GaussianCloud.empty(), grid, ctx=ctx)
    assert vol.shape == (8, 8, 8) and np.all(vol == 0.0)
    cloud = gsct.make_cloud("random", 4, seed=53)
    g = gsct.voxelize_backward(cloud, gsct.GridRegion.covering(gsct.GridSpec.centered((16, 16, 16), 1.0)),
                               np.zeros((16, 16, 16), np.float32), ctx=ctx)
    for k in ("positions", "log_scales", "rotations", "raw_densities"):
        assert np.all(getattr(g, k) == 0.0)


def test_homogeneity_and_determinism(ctx):
    """test_voxelizer.cpp:234-247"""
    cloud = gsct.make_cloud("random", 6, seed=58)
    grid = gsct.GridSpec.centered((20, 20, 20), 0.8)
    vs = gsct.VoxelSettings(tau_cut=1e-12)
    base = gsct.voxelize_full(cloud, grid, vs, ctx=ctx)
    twice = gsct.voxelize_full(gsct.GaussianCloud(cloud.positions, cloud.log_scales, cloud.rotations,
                                                  cloud.raw_densities * 2.0), grid, vs, ctx=ctx)
    assert np.array_equal(twice, 2.0 * base)
    assert np.array_equal(gsct.voxelize_full(cloud, grid, vs, ctx=ctx), base)


def test_region_matches_parent_window(ctx):
    """test_voxelizer.cpp:42-59 (fp32: agreement to rounding of the window origin)."""
    cloud = gsct.make_cloud("random", 6, seed=52, pos_range=4.0)
    grid = gsct.GridSpec.centered((24, 24, 24), 0.7)
    full = gsct.voxelize_full(cloud, grid, ctx=ctx)
    region = gsct.GridRegion.of_parent(grid, (5, 8, 2), (10, 9, 14))
    win = gsct.voxelize(cloud, region, ctx=ctx)
    sub = full[2:16, 8:17, 5:15]
    assert np.max(np.abs(win - sub)) <= 1e-5 * full.max()


def test_z_slabs_tile_full_volume_bitwise(ctx):
    """z-slab sharding: windows of the same grid reproduce the full volume bit for bit."""
    cloud = gsct.make_cloud("random", 80, seed=60, pos_range=6.0)
    grid = gsct.GridSpec.centered((30, 28, 37), 0.5)
    region = gsct.GridRegion.covering(grid)
    full = gsct.voxelize(cloud, region, ctx=ctx)
    cuts = [0, 9, 10, 24, 37]
    slabs = [gsct.voxelize(cloud, region, window=((0, 0, a), (30, 28, b)), ctx=ctx) for a, b in zip(cuts, cuts[1:])]
    assert np.array_equal(np.concatenate(slabs, axis=0), full)


def test_z_slab_backward_moments_sum(ctx, orc):
    """Backward under z-slab sharding: per-slab moments summed == full backward (tolerance)."""
    import torch

    cloud = gsct.make_cloud("random", 40, seed=61, pos_range=5.0)
    grid = gsct.GridSpec.centered((24, 24, 24), 0.6)
    region = gsct.GridRegion.covering(grid)
    gv = np.random.default_rng(3).uniform(-1, 1, size=(24, 24, 24)).astype(np.float32)
    full = gsct.voxelize_backward(cloud, region, gv, ctx=ctx)
    total = torch.zeros((10, cloud.size()), dtype=torch.float64, device="cuda")
    for a, b in ((0, 7), (7, 16), (16, 24)):
        m = torch.zeros_like(total)
        gsct.voxelize_backward_moments(cloud, region, torch.from_numpy(gv[a:b].copy()).cuda(),
                                       ((0, 0, a), (24, 24, b)), m, ctx=ctx)
        total += m
    g = gsct.voxelize_backward_finish(cloud, region, total, ctx=ctx)
    errs = grad_class_errors(g, {k: getattr(full, k) for k in ("positions", "log_scales", "rotations",
                                                               "raw_densities", "pos_grad_norm")})
    assert all(e <= 1e-5 for e in errs.values()), errs
    assert np.array_equal(g.visible, full.visible)


def test_voxel_contract_errors(ctx):
    cloud = gsct.make_cloud("random", 5, seed=2)
    cloud.log_scales[3, 2] = np.nan
    with pytest.raises(gsct.ContractError, match="non-finite parameter in splat 3"):
        gsct.voxelize_full(cloud, gsct.GridSpec.centered((8, 8, 8), 1.0), ctx=ctx)
    with pytest.raises(gsct.ContractError, match="grad dims"):
        gsct.voxelize_backward(gsct.make_cloud("random", 5, seed=2),
                               gsct.GridRegion.covering(gsct.GridSpec.centered((8, 8, 8), 1.0)),
                               np.zeros((8, 8, 7), np.float32), ctx=ctx)


@pytest.mark.parametrize("spacing", [0.25, 0.5, 2.0])
def test_peak_is_density_binary_spacings(ctx, spacing):
    """Exactly-on-lattice centres at power-of-two spacings, off-centre in the brick (the
    multiplicative x-chain must not be used for the peak row)."""
    grid = gsct.GridSpec.centered((21, 19, 23), spacing)
    origin = -0.5 * spacing * (np.array(grid.dims) - 1)
    idx = np.array([[3, 5, 7], [13, 9, 15], [18, 2, 20]])
    pos = origin + spacing * idx
    cloud = gsct.GaussianCloud(pos, np.full((3, 3), np.log(1.3 * spacing)), np.tile([1.0, 0, 0, 0], (3, 1)),
                               np.array([0.8, 1.7, 0.35]))
    vol = gsct.voxelize_full(cloud, grid, ctx=ctx)
    for (x, y, z), rho in zip(idx, (0.8, 1.7, 0.35)):
        assert vol[z, y, x] >= np.float32(rho)  # peak term exact; neighbours add >= 0


def test_forward_extreme_shapes(ctx, orc):
    """Needle splats (box corners underflow fp32 exp: the chain-safety fallback) and
    sub-voxel splats next to ordinary ones."""
    grid = gsct.GridSpec.centered((30, 28, 26), 0.5)
    base = gsct.make_cloud("random", 36, seed=61, pos_range=5.0)
    rng = np.random.default_rng(4)
    ls = base.log_scales.copy()
    ls[:12] = np.stack([np.full(12, -3.5), np.full(12, 0.9), np.full(12, -3.0)], axis=1)
    ls[12:24] = rng.uniform(-4.0, -2.5, size=(12, 3))
    cloud = gsct.GaussianCloud(base.positions, ls, base.rotations, base.raw_densities)
    region = gsct.GridRegion.covering(grid)
    vol = gsct.voxelize(cloud, region, gsct.VoxelSettings(), ctx=ctx)
    ref, _ = orc.voxelize(cloud, region, gsct.VoxelSettings())
    assert max_err_rel_peak(vol, ref) <= VOL_TOL
