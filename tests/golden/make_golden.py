"""Generates the golden fixtures in this directory from the REFERENCE itself
(oracle/_ref/libgsct_ref.so = /root/reference/proj/include/gsct/*.hpp compiled unchanged with
the test-only Eigen shim). Run where /root/reference exists:

    python tests/golden/make_golden.py

Each .npz holds the inputs (raw cloud parameters, geometry/grid, settings, upstream
gradients) and the reference outputs (per-splat integer boxes and flags, tile lists,
images/volumes in fp64, ParamGradients, RenderStats). The fixtures travel with the repo to
the GPU box, where /root/reference does not exist.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Ref  # noqa: E402
from paper_2604_01844_b200 import gsct  # noqa: E402

OUT = Path(__file__).resolve().parent


def cloud_dict(c):
    return dict(positions=c.positions, log_scales=c.log_scales, rotations=c.rotations, raw_densities=c.raw_densities)


def raster_case(ref, name, cloud, geom, rs, seed):
    h = ref.cloud(cloud)
    n = cloud.size()
    d = dict(cloud_dict(cloud))
    d.update(mode=geom.mode, n_u=geom.n_u, n_v=geom.n_v, s_u=geom.s_u, s_v=geom.s_v, angles=np.asarray(geom.angles),
             source_to_origin=geom.source_to_origin, origin_to_detector=geom.origin_to_detector,
             tau_cut=rs.tau_cut, sigma_cap=rs.sigma_cap, tile_size=rs.tile_size, dilate=rs.dilate,
             dilation_px2=rs.dilation_px2, bounding=rs.bounding)
    rng = np.random.default_rng(seed)
    for v in range(len(geom.angles)):
        pb = ref.project_and_bin(h, geom, v, rs, n)
        img, st = ref.rasterize_view(h, geom, v, rs)
        gi = rng.uniform(-1, 1, size=(geom.n_v, geom.n_u)).astype(np.float32).astype(np.float64)
        g = ref.rasterize_backward(h, geom, v, gi, rs, n)
        d.update({f"v{v}_rect": pb["rect"], f"v{v}_culled": pb["culled"], f"v{v}_degenerate": pb["degenerate"],
                  f"v{v}_tile_offsets": pb["tile_offsets"], f"v{v}_tile_splats": pb["tile_splats"],
                  f"v{v}_image": img, f"v{v}_grad_image": gi,
                  f"v{v}_stats": np.array([st["culled"], st["degenerate"], st["tile_pairs"], st["pixel_pairs"]])})
        for k in ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm", "visible"):
            d[f"v{v}_g_{k}"] = g[k]
    ref.free_cloud(h)
    np.savez_compressed(OUT / f"{name}.npz", **d)


def voxel_case(ref, name, cloud, region, vs, seed):
    h = ref.cloud(cloud)
    n = cloud.size()
    d = dict(cloud_dict(cloud))
    d.update(dims=np.asarray(region.dims), spacing=region.spacing, origin=np.asarray(region.origin),
             tau_cut=vs.tau_cut, sigma_cap=vs.sigma_cap)
    lo, hi, skip = ref.prepare_voxel_splats(h, region, vs, n)
    vol, st = ref.voxelize(h, region, vs)
    gv = np.random.default_rng(seed).uniform(-1, 1, size=vol.shape).astype(np.float32).astype(np.float64)
    g = ref.voxelize_backward(h, region, gv, vs, n)
    d.update(lo=lo, hi=hi, skip=skip, volume=vol, grad_volume=gv, stats=np.array([st["culled"], st["pixel_pairs"]]))
    for k in ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm", "visible"):
        d[f"g_{k}"] = g[k]
    ref.free_cloud(h)
    np.savez_compressed(OUT / f"{name}.npz", **d)


def main() -> None:
    ref = Ref()
    raster_case(ref, "raster_parallel_default", gsct.make_cloud("random", 20, seed=35),
                gsct.ScanGeometry("parallel", 52, 52, 0.55, 0.55, [2.4, 0.3]), gsct.RasterSettings(), 1)
    raster_case(ref, "raster_cone_oracle", gsct.make_cloud("random", 16, seed=42),
                gsct.ScanGeometry("cone", 40, 44, 0.7, 0.65, [0.9, 3.3], 50.0, 25.0),
                gsct.RasterSettings(tau_cut=1e-12, sigma_cap=6.0, dilate=False), 2)
    sl = gsct.make_cloud("shepp_logan", 1200, seed=0, side=64, spacing=1.0)
    sl_geom = gsct.default_geometry((64, 64, 64), 1.0, 75, "cone", 96, 96)
    sl_geom.angles = list(sl_geom.angles[::25])  # views 0, 25, 50 of the 75-view scan
    raster_case(ref, "raster_shepp_logan_cone", sl, sl_geom, gsct.RasterSettings(), 3)
    raster_case(ref, "raster_square_tile7", gsct.make_cloud("synthetic", 60, seed=21, scale=0.05, anisotropy=4.0,
                                                            density=0.5),
                gsct.ScanGeometry("parallel", 37, 33, 2.0 / 37, 2.0 / 33, [0.0, 1.2]),
                gsct.RasterSettings(bounding="square_circumscribed", tile_size=7), 4)
    grid = gsct.GridSpec.centered((20, 22, 18), 0.8)
    c = gsct.make_cloud("random", 16, seed=54, pos_range=4.0)
    c.raw_densities[3] = -0.2
    voxel_case(ref, "voxel_default", c, gsct.GridRegion.covering(grid), gsct.VoxelSettings(), 5)
    voxel_case(ref, "voxel_region_wide", c, gsct.GridRegion.of_parent(grid, (3, 2, 5), (9, 11, 7)),
               gsct.VoxelSettings(tau_cut=1e-12, sigma_cap=8.0), 6)
    voxel_case(ref, "voxel_shepp_logan", gsct.make_cloud("shepp_logan", 1000, seed=1, side=32, spacing=1.0),
               gsct.GridRegion.covering(gsct.GridSpec.centered((32, 32, 32), 1.0)), gsct.VoxelSettings(), 7)
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
