"""Pins the C restatement oracle (oracle/gsct_oracle.c) bit-for-bit against the UNCHANGED
reference compiled here (oracle/_ref/libgsct_ref.so, /root/reference/proj/include/gsct).

Covers every hot-path function of SURVEY.md 8(a): activation/covariance/projection/bbox
(project_cloud), bin_tiles, rasterize_view, rasterize_backward, prepare_voxel_splats,
voxelize, voxelize_backward — parallel and cone beams, default and oracle settings."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import cone_geometry, oracle_settings, parallel_geometry
from paper_2604_01844_b200 import gsct

CASES = [
    ("parallel-default", lambda: parallel_geometry(48, 0.6, [0.3, 2.0]), gsct.RasterSettings()),
    ("parallel-oracle", lambda: parallel_geometry(48, 0.6, [0.3, 2.0]), oracle_settings()),
    ("cone-default", lambda: cone_geometry(40, 0.7, [0.9, 4.0]), gsct.RasterSettings()),
    ("cone-oracle", lambda: cone_geometry(40, 0.7, [0.9, 4.0]), oracle_settings()),
    ("parallel-square-tile7", lambda: parallel_geometry(37, 0.5, [1.1]),
     gsct.RasterSettings(bounding="square_circumscribed", tile_size=7)),
]


@pytest.mark.parametrize("name,make_geom,rs", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("seed", [11, 42])
def test_raster_bitwise(orc, ref, name, make_geom, rs, seed):
    cloud = gsct.make_cloud("random", 24, seed=seed)
    geom = make_geom()
    h = ref.cloud(cloud)
    try:
        n = cloud.size()
        for view in range(len(geom.angles)):
            rp = ref.project_and_bin(h, geom, view, rs, n)
            op = orc.project_cloud(cloud, geom, view, rs)
            for k in ("rect", "culled", "degenerate", "mean2d", "conic", "amplitude"):
                assert np.array_equal(rp[k], op[k]), k
            off, vals = orc.bin_tiles(cloud, geom, view, rs)
            assert np.array_equal(off, rp["tile_offsets"])
            assert np.array_equal(vals, rp["tile_splats"])

            rimg, rst = ref.rasterize_view(h, geom, view, rs)
            oimg, ost = orc.rasterize_view(cloud, geom, view, rs)
            assert np.array_equal(rimg, oimg)
            for k in ("culled", "degenerate", "tile_pairs", "pixel_pairs"):
                assert rst[k] == ost[k], k

            rng = np.random.default_rng(seed + view)
            gi = rng.uniform(-1, 1, size=(geom.n_v, geom.n_u))
            gi[rng.uniform(size=gi.shape) < 0.1] = 0.0  # exercise the w == 0 skip
            rg = ref.rasterize_backward(h, geom, view, gi, rs, n)
            og = orc.rasterize_backward(cloud, geom, view, gi, rs)
            for k in ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm", "visible"):
                assert np.array_equal(rg[k], og[k]), k
    finally:
        ref.free_cloud(h)


VOX_CASES = [
    ("default", gsct.GridSpec.centered((20, 22, 18), 0.8), gsct.VoxelSettings()),
    ("wide", gsct.GridSpec.centered((16, 16, 16), 0.9), gsct.VoxelSettings(tau_cut=1e-12, sigma_cap=8.0)),
]


@pytest.mark.parametrize("name,grid,vs", VOX_CASES, ids=[c[0] for c in VOX_CASES])
def test_voxel_bitwise(orc, ref, name, grid, vs):
    cloud = gsct.make_cloud("random", 16, seed=54, pos_range=4.0)
    # push one density negative and one below tau to cover the clamp / skip branches
    cloud.raw_densities[3] = -0.2
    cloud.raw_densities[5] = 5e-5
    h = ref.cloud(cloud)
    try:
        n = cloud.size()
        for region in (gsct.GridRegion.covering(grid), gsct.GridRegion.of_parent(grid, (3, 2, 5), (9, 11, 7))):
            rlo, rhi, rskip = ref.prepare_voxel_splats(h, region, vs, n)
            olo, ohi, oskip = orc.prepare_voxel_splats(cloud, region, vs)
            assert np.array_equal(rskip, oskip)
            assert np.array_equal(rlo[~rskip], olo[~oskip]) and np.array_equal(rhi[~rskip], ohi[~oskip])
            rv, rst = ref.voxelize(h, region, vs)
            ov, ost = orc.voxelize(cloud, region, vs)
            assert np.array_equal(rv, ov)
            assert rst["culled"] == ost["culled"] and rst["pixel_pairs"] == ost["pixel_pairs"]
            gv = np.random.default_rng(7).uniform(-1, 1, size=rv.shape)
            rg = ref.voxelize_backward(h, region, gv, vs, n)
            og = orc.voxelize_backward(cloud, region, gv, vs)
            for k in ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm", "visible"):
                assert np.array_equal(rg[k], og[k]), k
    finally:
        ref.free_cloud(h)


def test_harness_generators_match_reference(ref):
    """synthetic_cloud (bench.hpp:33-52), oracles::random_cloud, default_geometry."""
    for aniso in (1.0, 10.0):
        p, l, q, r = ref.synthetic_cloud(64, anisotropy=aniso, density=0.02, scale=0.01, seed=21)
        c = gsct.make_cloud("synthetic", 64, seed=21, anisotropy=aniso, density=0.02, scale=0.01)
        for a, b in zip((p, l, q, r), (c.positions, c.log_scales, c.rotations, c.raw_densities)):
            assert np.array_equal(a, b)
    for seed, count, pr, lo, hi in ((11, 8, 5.0, 0.5, 2.5), (12, 8, 4.0, 0.15, 0.6), (300, 1, 5.0, 0.05, 10.0)):
        p, l, q, r = ref.random_cloud(seed, count, pr, lo, hi)
        c = gsct.make_cloud("random", count, seed=seed, pos_range=pr, scale_lo=lo, scale_hi=hi)
        for a, b in zip((p, l, q, r), (c.positions, c.log_scales, c.rotations, c.raw_densities)):
            assert np.array_equal(a, b)
    for cone in (0, 1):
        g, ang = ref.default_geometry((128, 96, 64), 0.5, 75, cone, 256, 200)
        gg = gsct.default_geometry((128, 96, 64), 0.5, 75, "cone" if cone else "parallel", 256, 200)
        assert (g.s_u, g.s_v, g.source_to_origin, g.origin_to_detector) == (
            gg.s_u, gg.s_v, gg.source_to_origin, gg.origin_to_detector)
        assert np.array_equal(ang, np.asarray(gg.angles))


def test_reference_arm_inputs_match_product_harness(ref):
    """bench.py's reference arm builds the C2 / C5 workloads without the product library
    (ref_shepp_logan_cloud with the reference Rng + default_geometry); they must be the
    very inputs our arm uses."""
    import bench

    for name in ("c1", "c2"):
        c_ours, g_ours = bench.make_workload(name)
        c_ref, g_ref = bench.make_workload_ref(ref, name)
        for a, b in zip((c_ref.positions, c_ref.log_scales, c_ref.rotations, c_ref.raw_densities),
                        (c_ours.positions, c_ours.log_scales, c_ours.rotations, c_ours.raw_densities)):
            assert np.array_equal(a, b)
        assert g_ref == g_ours or (
            (g_ref.mode, g_ref.n_u, g_ref.n_v, g_ref.s_u, g_ref.s_v, g_ref.source_to_origin, g_ref.origin_to_detector)
            == (g_ours.mode, g_ours.n_u, g_ours.n_v, g_ours.s_u, g_ours.s_v, g_ours.source_to_origin,
                g_ours.origin_to_detector) and np.array_equal(np.asarray(g_ref.angles), np.asarray(g_ours.angles)))
