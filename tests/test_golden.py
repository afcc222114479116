"""Golden fixtures produced by the reference itself (tests/golden/make_golden.py).

CPU: the restatement oracle reproduces every fixture bit for bit.
GPU: the CUDA path reproduces the integer outputs (boxes, flags, tile lists, RenderStats
counters) exactly, images/volumes within 1e-4 of peak and gradients within 1e-4 of the
per-class maximum (fp32 per-pair arithmetic vs the fp64 reference)."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from conftest import grad_class_errors, max_err_rel_peak
from paper_2604_01844_b200 import gsct

GOLDEN = Path(__file__).resolve().parent / "golden"
RASTER = sorted(p.stem for p in GOLDEN.glob("raster_*.npz"))
VOXEL = sorted(p.stem for p in GOLDEN.glob("voxel_*.npz"))
GRAD_KEYS = ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm")


def load(name):
    z = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    cloud = gsct.GaussianCloud(z["positions"], z["log_scales"], z["rotations"], z["raw_densities"])
    return z, cloud


def raster_inputs(z):
    geom = gsct.ScanGeometry(str(z["mode"]), int(z["n_u"]), int(z["n_v"]), float(z["s_u"]), float(z["s_v"]),
                             list(z["angles"]), float(z["source_to_origin"]), float(z["origin_to_detector"]))
    rs = gsct.RasterSettings(float(z["tau_cut"]), float(z["sigma_cap"]), int(z["tile_size"]), bool(z["dilate"]),
                             float(z["dilation_px2"]), str(z["bounding"]))
    return geom, rs


def voxel_inputs(z):
    region = gsct.GridRegion((0, 0, 0), tuple(int(d) for d in z["dims"]), float(z["spacing"]),
                             tuple(float(o) for o in z["origin"]))
    return region, gsct.VoxelSettings(float(z["tau_cut"]), float(z["sigma_cap"]))


def test_fixtures_present():
    assert len(RASTER) >= 4 and len(VOXEL) >= 3


@pytest.mark.parametrize("name", RASTER)
def test_oracle_reproduces_raster_golden(orc, name):
    z, cloud = load(name)
    geom, rs = raster_inputs(z)
    for v in range(len(geom.angles)):
        pc = orc.project_cloud(cloud, geom, v, rs)
        assert np.array_equal(pc["rect"][~pc["culled"]], z[f"v{v}_rect"][~z[f"v{v}_culled"]])
        assert np.array_equal(pc["culled"], z[f"v{v}_culled"]) and np.array_equal(pc["degenerate"], z[f"v{v}_degenerate"])
        off, vals = orc.bin_tiles(cloud, geom, v, rs)
        assert np.array_equal(off, z[f"v{v}_tile_offsets"]) and np.array_equal(vals, z[f"v{v}_tile_splats"])
        img, st = orc.rasterize_view(cloud, geom, v, rs)
        assert np.array_equal(img, z[f"v{v}_image"])
        assert [st["culled"], st["degenerate"], st["tile_pairs"], st["pixel_pairs"]] == z[f"v{v}_stats"].tolist()
        g = orc.rasterize_backward(cloud, geom, v, z[f"v{v}_grad_image"], rs)
        for k in GRAD_KEYS + ("visible",):
            assert np.array_equal(g[k], z[f"v{v}_g_{k}"]), k


@pytest.mark.parametrize("name", VOXEL)
def test_oracle_reproduces_voxel_golden(orc, name):
    z, cloud = load(name)
    region, vs = voxel_inputs(z)
    lo, hi, skip = orc.prepare_voxel_splats(cloud, region, vs)
    assert np.array_equal(skip, z["skip"])
    assert np.array_equal(lo[~skip], z["lo"][~skip]) and np.array_equal(hi[~skip], z["hi"][~skip])
    vol, st = orc.voxelize(cloud, region, vs)
    assert np.array_equal(vol, z["volume"]) and [st["culled"], st["pixel_pairs"]] == z["stats"].tolist()
    g = orc.voxelize_backward(cloud, region, z["grad_volume"], vs)
    for k in GRAD_KEYS + ("visible",):
        assert np.array_equal(g[k], z[f"g_{k}"]), k


@pytest.mark.gpu
@pytest.mark.parametrize("name", RASTER)
def test_gpu_matches_raster_golden(ctx, name):
    z, cloud = load(name)
    geom, rs = raster_inputs(z)
    st = gsct.RenderStats()
    imgs = gsct.rasterize_views(cloud, geom, None, rs, st, ctx=ctx)
    exp = np.zeros(4, dtype=np.int64)
    for v in range(len(geom.angles)):
        pc = gsct.project_cloud(cloud, geom, v, rs, ctx=ctx)
        vis = ~z[f"v{v}_culled"]
        assert np.array_equal(pc["culled"], z[f"v{v}_culled"]) and np.array_equal(pc["degenerate"], z[f"v{v}_degenerate"])
        assert np.array_equal(pc["rect"][vis], z[f"v{v}_rect"][vis])
        keys, vals = gsct.tile_pairs(cloud, geom, [v], rs, ctx=ctx)
        off = z[f"v{v}_tile_offsets"]
        assert np.array_equal(keys, np.repeat(np.arange(len(off) - 1), np.diff(off)).astype(np.uint32))
        assert np.array_equal(vals.astype(np.int32), z[f"v{v}_tile_splats"])
        assert max_err_rel_peak(imgs[v], z[f"v{v}_image"]) <= 1e-4
        exp += z[f"v{v}_stats"]
    assert [st.culled, st.degenerate, st.tile_pairs, st.pixel_pairs] == exp.tolist()
    gi = np.stack([z[f"v{v}_grad_image"] for v in range(len(geom.angles))]).astype(np.float32)
    g = gsct.rasterize_backward_views(cloud, geom, None, gi, rs, ctx=ctx)
    ref = {k: sum(z[f"v{v}_g_{k}"] for v in range(len(geom.angles))) for k in GRAD_KEYS}
    errs = grad_class_errors(g, ref)
    assert all(e <= 1e-4 for e in errs.values()), errs
    vis = np.zeros_like(z["v0_g_visible"])
    for v in range(len(geom.angles)):
        vis |= z[f"v{v}_g_visible"]
    assert np.array_equal(g.visible, vis)


@pytest.mark.gpu
@pytest.mark.parametrize("name", VOXEL)
def test_gpu_matches_voxel_golden(ctx, name):
    z, cloud = load(name)
    region, vs = voxel_inputs(z)
    lo, hi, skip = gsct.voxel_boxes(cloud, region, vs, ctx=ctx)
    assert np.array_equal(skip, z["skip"])
    assert np.array_equal(lo[~skip], z["lo"][~skip]) and np.array_equal(hi[~skip], z["hi"][~skip])
    st = gsct.RenderStats()
    vol = gsct.voxelize(cloud, region, vs, st, ctx=ctx)
    assert max_err_rel_peak(vol, z["volume"]) <= 1e-4
    assert [st.culled, st.pixel_pairs] == z["stats"].tolist()
    g = gsct.voxelize_backward(cloud, region, z["grad_volume"].astype(np.float32), vs, ctx=ctx)
    errs = grad_class_errors(g, {k: z[f"g_{k}"] for k in GRAD_KEYS})
    assert all(e <= 1e-4 for e in errs.values()), errs
    assert np.array_equal(g.visible, z["g_visible"])
