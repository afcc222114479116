"""The C restatement oracle against the reference tests' known answers and independent
re-derivations (tests/oracles.hpp): integer bbox golden values, line-integral factor,
ray quadrature, direct field sums, central finite differences. CPU only, seconds."""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import cone_geometry, max_err_rel_peak, oracle_settings, parallel_geometry
from paper_2604_01844_b200 import gsct


def test_splat_bbox_known_answers(orc):
    """test_projector.cpp:122-145"""
    ok, _ = orc.splat_bbox(1e-5, np.eye(2), [16, 16], 1e-4, 64, 64)
    assert not ok
    ok, r = orc.splat_bbox(math.exp(4.5) * 1e-4, 4.0 * np.eye(2), [32, 32], 1e-4, 64, 64)
    assert ok and r == [26, 38, 26, 38]
    ok, r = orc.splat_bbox(math.exp(2.0) * 1e-4, np.diag([100.0, 1.0]), [64, 64], 1e-4, 128, 128)
    assert ok and r == [44, 84, 62, 66]


def test_splat_bbox_contains_everything_above_cutoff(orc):
    """test_projector.cpp:147-175"""
    rng = gsct.Rng(17)
    uu, vv = np.meshgrid(np.arange(64), np.arange(64))
    for _ in range(30):
        a, c = rng.uniform(0.5, 40.0), rng.uniform(0.5, 40.0)
        b = rng.uniform(-0.9, 0.9) * math.sqrt(a * c)
        cov = np.array([[a, b], [b, c]])
        mean = np.array([rng.uniform(20, 44), rng.uniform(20, 44)])
        g = 1e-4 * math.exp(rng.uniform(0.5, 4.0))
        ok, r = orc.splat_bbox(g, cov, mean, 1e-4, 64, 64)
        if not ok:
            continue
        conic = np.linalg.inv(cov)
        d = np.stack([uu - mean[0], vv - mean[1]], -1)
        val = g * np.exp(-0.5 * np.einsum("...i,ij,...j", d, conic, d))
        above = val > 1e-4
        assert np.all(uu[above] >= r[0]) and np.all(uu[above] <= r[1])
        assert np.all(vv[above] >= r[2]) and np.all(vv[above] <= r[3])


def one(pos, ls, q, rho) -> gsct.GaussianCloud:
    return gsct.GaussianCloud(np.array([pos], float), np.array([ls], float), np.array([q], float), np.array([rho]))


def test_line_integral_factor(orc):
    """test_projector.cpp:69-92: mu = sqrt(2 pi) * s for isotropic splats, any rotation."""
    geom = parallel_geometry(32, 1.0, [0.4])
    pc = orc.project_cloud(one([0, 0, 0], [0, 0, 0], [1, 0, 0, 0], 1.0), geom, 0, oracle_settings())
    assert pc["amplitude"][0] == pytest.approx(math.sqrt(2 * math.pi), rel=1e-12)
    rng = gsct.Rng(3)
    geom = parallel_geometry(32, 1.0, [1.1])
    for s in (0.3, 1.7, 4.2):
        for _ in range(5):
            q = np.array([rng.normal() for _ in range(4)])
            q /= np.linalg.norm(q)
            pc = orc.project_cloud(one([0, 0, 0], [math.log(s)] * 3, q, 1.0), geom, 0, oracle_settings())
            assert pc["amplitude"][0] == pytest.approx(math.sqrt(2 * math.pi) * s, rel=1e-10)


def _quadrature_image(cloud, geom, view):
    """oracles.hpp:23-44 + test_projector.cpp:31-49 (midpoint quadrature along each ray)."""
    f = gsct.view_frame(geom, view)
    img = np.zeros((geom.n_v, geom.n_u))
    cu, cv = 0.5 * (geom.n_u - 1), 0.5 * (geom.n_v - 1)
    uu, vv = np.meshgrid(np.arange(geom.n_u), np.arange(geom.n_v))
    pix = (f["detector_center"][None, None, :] + ((uu - cu) * geom.s_u)[..., None] * f["u"]
           + ((vv - cv) * geom.s_v)[..., None] * f["v"])
    if f["cone"]:
        origin = np.broadcast_to(f["source"], pix.shape)
        d = pix - f["source"]
        dirs = d / np.linalg.norm(d, axis=-1, keepdims=True)
    else:
        origin = pix
        dirs = np.broadcast_to(f["d"], pix.shape)
    for i in range(cloud.size()):
        s = np.exp(cloud.log_scales[i])
        q = cloud.rotations[i] / np.linalg.norm(cloud.rotations[i])
        w, x, y, z = q
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                      [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                      [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
        sig = R @ np.diag(s * s) @ R.T
        A = np.linalg.inv(sig)
        p = cloud.positions[i]
        rho = max(cloud.raw_densities[i], 0.0)
        beta = np.einsum("...i,ij,...j", dirs, A, dirs)
        wv = origin - p
        t_star = -np.einsum("...i,ij,...j", wv, A, dirs) / beta
        sr = 1.0 / np.sqrt(beta)
        smin = math.sqrt(np.linalg.eigvalsh(sig).min())
        step = smin / 20.0
        t0, t1 = t_star - 6 * sr, t_star + 6 * sr
        n = np.ceil((t1 - t0) / step).astype(int)
        nmax = int(n.max())
        k = np.arange(nmax)
        dt = (t1 - t0) / n
        t = t0[..., None] + (k + 0.5) * dt[..., None]
        xs = origin[..., None, :] + t[..., None] * dirs[..., None, :] - p
        vals = np.exp(-0.5 * np.einsum("...i,ij,...j", xs, A, xs)) * (k < n[..., None])
        img += rho * vals.sum(-1) * dt
    return img


def test_parallel_projection_matches_quadrature(orc):
    """test_projector.cpp:94-102 (<= 1e-3 of peak)"""
    cloud = gsct.make_cloud("random", 8, seed=11)
    geom = parallel_geometry(48, 0.6, [0.3, 2.0])
    for view in range(2):
        img, _ = orc.rasterize_view(cloud, geom, view, oracle_settings())
        assert max_err_rel_peak(img, _quadrature_image(cloud, geom, view)) < 1e-3


def test_cone_projection_matches_quadrature_small_splats(orc):
    """test_projector.cpp:104-120 (<= 5% of peak)"""
    cloud = gsct.make_cloud("random", 8, seed=12, pos_range=4.0, scale_lo=0.15, scale_hi=0.6)
    geom = gsct.ScanGeometry("cone", 48, 48, 0.7, 0.7, [0.9], 60.0, 30.0)
    img, _ = orc.rasterize_view(cloud, geom, 0, oracle_settings())
    assert max_err_rel_peak(img, _quadrature_image(cloud, geom, 0)) < 0.05


def test_voxelize_matches_direct_field_sum(orc):
    """test_voxelizer.cpp:24-40 / acceptance criterion 3 (<= 1e-4 of peak) + peak == rho."""
    cloud = gsct.make_cloud("random", 12, seed=51, pos_range=6.0)
    grid = gsct.GridSpec.centered((32, 32, 32), 0.55)
    vol, _ = orc.voxelize(cloud, gsct.GridRegion.covering(grid), gsct.VoxelSettings(tau_cut=1e-12, sigma_cap=6.0))
    ax = [grid.origin[a] + grid.spacing * np.arange(grid.dims[a]) for a in range(3)]
    Z, Y, X = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    pts = np.stack([X, Y, Z], -1)
    ref = np.zeros(X.shape)
    for i in range(cloud.size()):
        s = np.exp(cloud.log_scales[i])
        w, x, y, z = cloud.rotations[i] / np.linalg.norm(cloud.rotations[i])
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                      [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                      [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
        A = np.linalg.inv(R @ np.diag(s * s) @ R.T)
        d = pts - cloud.positions[i]
        ref += max(cloud.raw_densities[i], 0.0) * np.exp(-0.5 * np.einsum("...i,ij,...j", d, A, d))
    assert max_err_rel_peak(vol, ref) <= 1e-4
    peak, _ = orc.voxelize(one([0, 0, 0], [math.log(1.5)] * 3, [1, 0, 0, 0], 0.8),
                           gsct.GridRegion.covering(gsct.GridSpec.centered((9, 9, 9), 1.0)), gsct.VoxelSettings())
    assert peak[4, 4, 4] == 0.8


def _fd(f, x0, h):
    return (f(x0 + h) - f(x0 - h)) / (2 * h)


@pytest.mark.parametrize("mode", ["parallel", "cone"])
def test_raster_backward_matches_finite_differences(orc, mode):
    """test_projector.cpp:327-364 (rel <= 1e-3, all four parameter classes)."""
    cloud = gsct.make_cloud("random", 4, seed=41 if mode == "parallel" else 42)
    geom = (parallel_geometry(36, 0.7, [0.9]) if mode == "parallel" else cone_geometry(36, 0.7, [0.9]))
    rs = oracle_settings()
    gi = np.random.default_rng(99).uniform(-1, 1, size=(36, 36))
    g = orc.rasterize_backward(cloud, geom, 0, gi, rs)

    def loss():
        return float(np.sum(orc.rasterize_view(cloud, geom, 0, rs)[0] * gi))

    worst = 0.0
    for name, arr in (("positions", cloud.positions), ("log_scales", cloud.log_scales),
                      ("rotations", cloud.rotations)):
        for i in range(cloud.size()):
            for a in range(arr.shape[1]):
                x0 = arr[i, a]
                h = max(abs(x0) * 1e-5, 1e-7)
                arr[i, a] = x0 + h
                fp = loss()
                arr[i, a] = x0 - h
                fm = loss()
                arr[i, a] = x0
                fd = (fp - fm) / (2 * h)
                an = g[name][i, a]
                if abs(fd) <= 1e-6 and abs(an) <= 1e-6:
                    continue
                worst = max(worst, abs(fd - an) / max(abs(fd), abs(an), 1e-9))
    assert worst < 1e-3


def test_voxel_backward_matches_finite_differences(orc):
    """test_voxelizer.cpp:74-104"""
    cloud = gsct.make_cloud("random", 3, seed=54, pos_range=4.0)
    grid = gsct.GridSpec.centered((20, 20, 20), 0.8)
    region = gsct.GridRegion.covering(grid)
    vs = gsct.VoxelSettings(tau_cut=1e-12, sigma_cap=8.0)
    gv = np.random.default_rng(7).uniform(-1, 1, size=(20, 20, 20))
    g = orc.voxelize_backward(cloud, region, gv, vs)

    def loss():
        return float(np.sum(orc.voxelize(cloud, region, vs)[0] * gv))

    worst = 0.0
    for name, arr in (("positions", cloud.positions), ("log_scales", cloud.log_scales),
                      ("rotations", cloud.rotations), ("raw_densities", cloud.raw_densities.reshape(-1, 1))):
        for i in range(cloud.size()):
            for a in range(arr.shape[1]):
                x0 = arr[i, a]
                h = max(abs(x0) * 1e-5, 1e-7)
                arr[i, a] = x0 + h
                fp = loss()
                arr[i, a] = x0 - h
                fm = loss()
                arr[i, a] = x0
                fd = (fp - fm) / (2 * h)
                an = g[name][i] if name == "raw_densities" else g[name][i, a]
                if abs(fd) <= 1e-6 and abs(an) <= 1e-6:
                    continue
                worst = max(worst, abs(fd - an) / max(abs(fd), abs(an), 1e-9))
    assert worst < 1e-3


def test_bin_tiles_known_answer(orc):
    """test_projector.cpp:270-289: two splats, 2x2 tiles of 16 px -> pair_count 5."""
    # a tiny parallel scene whose two splats land exactly on the reference's rectangles is
    # awkward to construct; use the oracle's bin_tiles directly on the C splat records
    import ctypes as C

    from oracle.oracle import _Splat

    arr = (_Splat * 2)()
    arr[0].culled = 0
    arr[0].u_min, arr[0].u_max, arr[0].v_min, arr[0].v_max = 2, 9, 3, 8
    arr[1].culled = 0
    arr[1].u_min, arr[1].u_max, arr[1].v_min, arr[1].v_max = 12, 20, 10, 18
    off = np.zeros(5, dtype=np.int64)
    pairs = orc.l.orc_bin_tiles(C.c_int64(2), arr, 32, 32, 16, C.c_void_p(off.ctypes.data), None)
    assert pairs == 5
    assert np.diff(off).tolist() == [2, 1, 1, 1]
