"""Next-row operators: the fused L1 + SSIM2D image loss and device Adam.

CPU part (not gpu): the oracle for both is the UNCHANGED reference compiled here
(oracle/_ref: losses.hpp total_loss_recon, optim.hpp adam_step; its own test_losses passes,
test_reference_suite.py). Here the reference loss is further pinned against an independent
brute-force numpy SSIM (every 11x11 window summed directly) and central differences.
GPU part: the CUDA operators through the C ABI against that reference:
  * image loss: per-view l1 / ssim / total within 1e-6 relative, gradient max|d| <= 1e-5 of
    the max |g_ref| (fp32 images and gradient, fp64 moments);
  * Adam: bit-identical parameters and moments after several steps (incl. a non-finite
    gradient that must be skipped and a density clamped at 0)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2604_01844_b200 import gsct


def _brute_ssim_loss(p: np.ndarray, t: np.ndarray) -> float:
    d = np.arange(11) - 5.0
    w1 = np.exp(-0.5 * d * d / 2.25)
    w1 /= w1.sum()
    w = np.outer(w1, w1)
    nv, nu = p.shape
    vals = []
    for y in range(nv - 10):
        for x in range(nu - 10):
            a, b = p[y:y + 11, x:x + 11], t[y:y + 11, x:x + 11]
            mx, my = (w * a).sum(), (w * b).sum()
            sx = (w * a * a).sum() - mx * mx
            sy = (w * b * b).sum() - my * my
            sxy = (w * a * b).sum() - mx * my
            vals.append((2 * mx * my + 1e-4) * (2 * sxy + 9e-4) / ((mx * mx + my * my + 1e-4) * (sx + sy + 9e-4)))
    return 1.0 - float(np.mean(vals))


def test_reference_loss_pinned_by_brute_force_and_fd(ref):
    rng = np.random.default_rng(0)
    p = rng.uniform(0, 1, size=(17, 19))
    t = np.clip(p + rng.normal(0, 0.1, size=p.shape), 0, 1)
    (l1, ssim, total), g = ref.total_loss_recon(p, t, 0.25)
    assert abs(l1 - np.mean(np.abs(p - t))) < 1e-14
    assert abs(ssim - _brute_ssim_loss(p, t)) < 1e-12
    assert abs(total - (l1 + 0.25 * ssim)) < 1e-14
    # central differences of the total at a few pixels away from |p - t| kinks
    for (y, x) in [(3, 4), (8, 9), (16, 18), (0, 0)]:
        if abs(p[y, x] - t[y, x]) < 1e-3:
            continue
        h = 1e-6
        pp, pm = p.copy(), p.copy()
        pp[y, x] += h
        pm[y, x] -= h
        fd = (ref.total_loss_recon(pp, t, 0.25)[0][2] - ref.total_loss_recon(pm, t, 0.25)[0][2]) / (2 * h)
        assert abs(fd - g[y, x]) <= 1e-6 * max(1.0, abs(g[y, x])) + 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(3, 48, 64), (2, 11, 11), (1, 70, 45)])
def test_image_loss_matches_reference(ref, ctx, shape):
    import torch
    rng = np.random.default_rng(sum(shape))
    p = rng.uniform(0, 1, size=shape).astype(np.float32)
    t = np.clip(p + rng.normal(0, 0.15, size=shape), 0, 1).astype(np.float32)
    t[0, :3, :3] = p[0, :3, :3]  # exact ties: sign(0) = 0
    for dev in (False, True):
        pi = torch.from_numpy(p).cuda() if dev else p
        ti = torch.from_numpy(t).cuda() if dev else t
        losses, grad = gsct.image_loss(pi, ti, 0.25, ctx=ctx)
        grad = grad.cpu().numpy() if dev else grad
        for v in range(shape[0]):
            want, gref = ref.total_loss_recon(p[v].astype(np.float64), t[v].astype(np.float64), 0.25)
            np.testing.assert_allclose(losses[v], want, rtol=1e-6, atol=1e-9)
            assert np.max(np.abs(grad[v] - gref)) <= 1e-5 * np.max(np.abs(gref))


@pytest.mark.gpu
def test_image_loss_contract(ctx):
    a = np.zeros((1, 10, 40), dtype=np.float32)
    with pytest.raises(gsct.ContractError, match="11x11"):
        gsct.image_loss(a, a, 0.25, ctx=ctx)


@pytest.mark.gpu
def test_adam_step_bit_identical(ref, ctx):
    import torch
    n = 257
    cloud = gsct.make_cloud("random", n, seed=5)
    cloud.raw_densities[:5] = 1e-7  # pushed below 0 by the update -> clamped
    rng = np.random.default_rng(1)
    host = {"pos": cloud.positions.copy(), "ls": cloud.log_scales.copy(), "q": cloud.rotations.copy(),
            "raw": cloud.raw_densities.copy()}
    keys = ("m_pos", "v_pos", "m_ls", "v_ls", "m_rot", "v_rot", "m_dens", "v_dens")
    shapes = {"m_pos": (n, 3), "v_pos": (n, 3), "m_ls": (n, 3), "v_ls": (n, 3), "m_rot": (n, 4), "v_rot": (n, 4),
              "m_dens": (n,), "v_dens": (n,)}
    hm = {k: np.zeros(shapes[k]) for k in keys}
    dcloud = cloud.to_device(0)
    st = gsct.AdamState(n, 0)
    lrs = gsct.LearningRates()
    step = skipped = 0
    for it in range(4):
        g = {"pos": rng.normal(size=(n, 3)), "ls": rng.normal(size=(n, 3)), "q": rng.normal(size=(n, 4)),
             "raw": np.abs(rng.normal(size=n)) * 1e3}
        if it == 2:
            g["q"][7, 1] = np.nan
            g["pos"][9, 0] = np.inf
        dg = gsct.ParamGradients(*[torch.from_numpy(np.ascontiguousarray(g[k])).cuda() for k in ("pos", "ls", "q", "raw")],
                                 torch.zeros(n, dtype=torch.float64, device="cuda"),
                                 torch.zeros(n, dtype=torch.uint8, device="cuda"))
        gsct.adam_step(dcloud, st, dg, lrs, ctx=ctx)
        step, skipped = ref.adam_step(host, hm, g, lrs, step, skipped)
    assert st.step == step == 4 and st.skipped_updates == skipped == 2
    got = dcloud.numpy()
    for a, k in ((got.positions, "pos"), (got.log_scales, "ls"), (got.rotations, "q"), (got.raw_densities, "raw")):
        assert np.array_equal(a, host[k]), k
    assert np.all(got.raw_densities >= 0.0) and np.any(got.raw_densities[:5] == 0.0)
    for k in keys:
        assert np.array_equal(getattr(st, k).cpu().numpy(), hm[k]), k


def test_reference_ssim3d_paths_and_tv_fd(ref):
    """The reference's streaming and materialised SSIM3D agree bit for bit
    (test_losses.cpp:140-149); TV3D gradient vs central differences."""
    rng = np.random.default_rng(2)
    v = rng.uniform(0, 1, size=(12, 13, 14))
    t = np.clip(v + rng.normal(0, 0.1, size=v.shape), 0, 1)
    a, ga = ref.total_loss_fit(v, t, 0.2, streaming=True)
    b, gb = ref.total_loss_fit(v, t, 0.2, streaming=False)
    assert np.array_equal(a, b) and np.array_equal(ga, gb)
    val, g = ref.tv3d(v)
    for idx in [(3, 4, 5), (0, 0, 0), (11, 12, 13)]:
        h = 1e-6
        vp, vm = v.copy(), v.copy()
        vp[idx] += h
        vm[idx] -= h
        fd = (ref.tv3d(vp)[0] - ref.tv3d(vm)[0]) / (2 * h)
        assert abs(fd - g[idx]) <= 1e-6 * max(1.0, abs(g[idx]))


@pytest.mark.gpu
@pytest.mark.parametrize("shape,alpha", [((12, 13, 14), 0.2), ((20, 11, 16), 0.5), ((5, 6, 7), 0.0)])
def test_volume_loss_matches_reference(ref, ctx, shape, alpha):
    import torch
    rng = np.random.default_rng(sum(shape))
    v = rng.uniform(0, 1, size=shape).astype(np.float32)
    t = np.clip(v + rng.normal(0, 0.1, size=shape), 0, 1).astype(np.float32)
    want, gref = ref.total_loss_fit(v.astype(np.float64), t.astype(np.float64), alpha)
    for dev in (False, True):
        vi = torch.from_numpy(v).cuda() if dev else v
        ti = torch.from_numpy(t).cuda() if dev else t
        got, g = gsct.volume_loss(vi, ti, alpha, ctx=ctx)
        g = g.cpu().numpy() if dev else g
        np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-9)
        assert np.max(np.abs(g - gref)) <= 1e-5 * np.max(np.abs(gref))


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(32, 32, 32), (2, 3, 4), (9, 17, 5)])
def test_tv3d_matches_reference(ref, ctx, shape):
    rng = np.random.default_rng(len(shape) + shape[0])
    v = rng.uniform(0, 1, size=shape).astype(np.float32)
    val, g = gsct.tv3d(v, ctx=ctx)
    rv, rg = ref.tv3d(v.astype(np.float64))
    assert abs(val - rv) <= 1e-9 * max(1.0, abs(rv))
    assert np.max(np.abs(g - rg)) <= 1e-6 * np.max(np.abs(rg))


@pytest.mark.gpu
@pytest.mark.parametrize("cone", [False, True])
def test_raymarch_matches_reference(ref, ctx, cone):
    """raymarch_project (synthetic.hpp:171-232) vs the reference on a random volume:
    fp64 rays and sums, fp32 trilinear weights/values -> within 1e-6 of the peak."""
    import torch
    dims = (23, 19, 17)  # x, y, z
    sp = 0.8
    grid = gsct.GridSpec.centered(dims, sp)
    rng = np.random.default_rng(11)
    vol = rng.uniform(0, 1, size=(dims[2], dims[1], dims[0])).astype(np.float32)
    if cone:
        geom = gsct.ScanGeometry("cone", 40, 36, 0.9, 0.8, [0.0, 0.7, 2.9, np.pi / 2], 60.0, 30.0)
    else:
        geom = gsct.ScanGeometry("parallel", 40, 36, 0.6, 0.55, [0.0, 0.4, 1.7, np.pi / 2], 0.0, 0.0)
    want = ref.raymarch_project(vol.astype(np.float64), sp, grid.origin, geom)
    got = gsct.raymarch_project(vol, grid, geom, ctx=ctx)
    assert np.max(np.abs(got - want)) <= 1e-6 * np.max(np.abs(want))
    gd = gsct.raymarch_project(torch.from_numpy(vol).cuda(), grid, geom, ctx=ctx).cpu().numpy()
    assert np.array_equal(gd, got)


def test_lr_schedule_and_scene_extent():
    """lr_schedule (optim.hpp:71-78) and scene_extent (core.hpp:120-129) of the host mirror:
    log-linear decay clamped at the ends, contract on non-positive rates; half the diagonal
    of the positions' bounding box."""
    base, final, horizon = 2e-4 * 7.5, 1e-6 * 7.5, 22500
    assert gsct.lr_schedule(base, final, 0, horizon) == base
    assert gsct.lr_schedule(base, final, -3, horizon) == base
    assert gsct.lr_schedule(base, final, horizon, horizon) == final
    assert gsct.lr_schedule(base, final, 10 * horizon, horizon) == final
    assert gsct.lr_schedule(base, final, 5, 0) == final
    mid = gsct.lr_schedule(base, final, horizon // 2, horizon)
    assert mid == pytest.approx(base * (final / base) ** ((horizon // 2) / horizon), rel=1e-15)
    assert final < mid < base
    with pytest.raises(gsct.ContractError):
        gsct.lr_schedule(0.0, final, 1, horizon)
    cloud = gsct.make_cloud("random", 500, seed=4, pos_range=3.0)
    p = np.asarray(cloud.positions)
    assert gsct.scene_extent(cloud) == pytest.approx(0.5 * np.linalg.norm(p.max(0) - p.min(0)), rel=1e-15)
    with pytest.raises(gsct.ContractError):
        gsct.scene_extent(gsct.GaussianCloud.empty())
