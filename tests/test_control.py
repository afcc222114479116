"""Adaptive density control: accumulate_control_stats
(optim.hpp:366-373) and adaptive_control (optim.hpp:201-317).

Oracle: the UNCHANGED reference compiled here (oracle/_ref, its own test_optim runs in
test_reference_suite.py). CPU part: the reference pinned against an independent numpy
restatement of the decisions (prune threshold, eligibility, the max_gaussians budget in
index order, clone vs split) and of the splice order; the engine state is unchanged by
the call (the reference draws the split children from state.rng and then replaces the state
with a copy taken before the draws, optim.hpp:244, 301, 315). GPU part: the device operator through the C ABI against the reference:
report, output size, which rows are copies / fresh, copied rows and all moments bit-exact,
the engine state unchanged, split-children positions within 1e-12 relative
(CUDA log/cos vs glibc, <= 2 ulp), clone nudges within 1e-13 relative."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2604_01844_b200 import gsct

KEYS = ("m_pos", "v_pos", "m_ls", "v_ls", "m_rot", "v_rot", "m_dens", "v_dens")
WIDTH = {"m_pos": 3, "v_pos": 3, "m_ls": 3, "v_ls": 3, "m_rot": 4, "v_rot": 4, "m_dens": 1, "v_dens": 1}


def _scene_extent(pos: np.ndarray) -> float:
    """core.hpp:120-129"""
    d = pos.max(axis=0) - pos.min(axis=0)
    return 0.5 * float(np.sqrt(d @ d))


def _case(kind: str, seed: int = 0):
    """(params, moments, acc, config dict, rng seed, draws consumed before the call)."""
    rng = np.random.default_rng(seed)
    if kind == "mixed":
        n = 3000
        c = gsct.make_cloud("random", n, seed=seed + 11)
    else:
        n = 64
        c = gsct.make_cloud("random", n, seed=seed + 3)
    p = {"pos": c.positions.copy(), "ls": c.log_scales.copy(), "q": c.rotations.copy(), "raw": c.raw_densities.copy()}
    mom = {k: rng.normal(size=(n, WIDTH[k]) if WIDTH[k] > 1 else (n,)) for k in KEYS}
    acc = {"grad_norm": np.zeros(n), "grad_dir": np.zeros((n, 3)), "count": np.zeros(n, dtype=np.int64)}
    cfg = dict(grad_threshold=5e-5, prune_density=5e-4, split_scale_fraction=0.01,
               scene_extent=_scene_extent(p["pos"]), max_gaussians=100000)
    pre_draws = 0
    if kind == "prune":
        p["raw"][[2, 17, 40]] = 0.0
        p["raw"][5] = -0.25  # activated density 0 too
    elif kind in ("split", "clone", "cap", "mixed", "many_splits"):
        acc["count"][:] = rng.integers(0, 4, size=n)
        acc["grad_norm"][:] = rng.uniform(0, 2e-4, size=n) * acc["count"]
        acc["grad_dir"][:] = rng.normal(size=(n, 3))
        acc["grad_dir"][::7] = 0.0  # zero direction: the clone is not nudged
        if kind == "clone":
            cfg["scene_extent"] = 1e3  # everything is small: clones only
        if kind == "split":
            cfg["scene_extent"] = 1e-3  # everything is large: splits only
            pre_draws = 100  # the engine mid-block
        if kind == "cap":
            cfg["max_gaussians"] = n + 9
        if kind == "mixed":
            p["raw"][rng.random(n) < 0.05] = 0.0
            p["ls"][rng.random(n) < 0.3] += 3.0  # a share of large splats: both clones and splits
            cfg["max_gaussians"] = n + 700
            cfg["scene_extent"] = 25.0
            pre_draws = 311
        if kind == "many_splits":
            acc["count"][:] = 1
            acc["grad_norm"][:] = 1.0
            cfg["scene_extent"] = 1e-3
            pre_draws = 5
    return p, mom, acc, cfg, 1234 + seed, pre_draws


def _rng_state(seed: int, pre_draws: int) -> np.ndarray:
    r = gsct.Rng(seed)
    for _ in range(pre_draws):
        r.uniform()
    st = r.state()
    return np.array(list(st.x) + [st.p], dtype=np.uint64)


def _numpy_decisions(p, acc, cfg):
    """Independent restatement of optim.hpp:207-241: op per splat (0 keep, 1 prune,
    2 clone, 3 split)."""
    density = np.maximum(p["raw"], 0.0)
    prune_below = cfg["prune_density"] * density.max()
    ops = np.where(density < prune_below, 1, 0)
    survivors = int((ops == 0).sum())
    budget = cfg["max_gaussians"] - survivors
    for i in range(len(ops)):
        if budget <= 0:
            break
        if ops[i] != 0 or acc["count"][i] == 0:
            continue
        if acc["grad_norm"][i] / float(acc["count"][i]) <= cfg["grad_threshold"]:
            continue
        ops[i] = 2 if np.exp(p["ls"][i]).max() < cfg["split_scale_fraction"] * cfg["scene_extent"] else 3
        budget -= 1
    return ops


CASES = ["calm", "prune", "split", "clone", "cap", "mixed", "many_splits"]


@pytest.mark.parametrize("kind", CASES)
def test_reference_control_pinned_by_numpy_restatement(ref, kind):
    p, mom, acc, cfg, seed, pre = _case(kind)
    st = _rng_state(seed, pre)
    st0 = st.copy()
    op, om, rep = ref.adaptive_control(p, mom, acc, st, **cfg)
    ops = _numpy_decisions(p, acc, cfg)
    assert rep["pruned"] == int((ops == 1).sum())
    assert rep["cloned"] == int((ops == 2).sum())
    assert rep["split"] == int((ops == 3).sum())
    assert rep["n_next"] == int((ops == 0).sum() + 2 * ((ops == 2) | (ops == 3)).sum())
    assert rep["n_next"] <= max(len(ops), cfg["max_gaussians"])
    # splice order: keep -> copy; clone -> copy + fresh; split -> two fresh rows
    r = 0
    for i, o in enumerate(ops):
        if o == 1:
            continue
        if o in (0, 2):
            assert np.array_equal(op["pos"][r], p["pos"][i]) and np.array_equal(om["m_pos"][r], mom["m_pos"][i])
            r += 1
        if o == 2:
            assert np.array_equal(op["ls"][r], p["ls"][i]) and not om["v_rot"][r].any()
            r += 1
        if o == 3:
            for _ in range(2):
                assert np.allclose(op["ls"][r], p["ls"][i] - np.log(1.6), rtol=0, atol=1e-15)
                assert op["raw"][r] == p["raw"][i] and not om["m_pos"][r].any()
                r += 1
    assert r == rep["n_next"]
    # the engine state is unchanged: the children draw from state.rng, then the state is
    # replaced by next_state, copied before the draws (optim.hpp:244, 301, 315)
    assert np.array_equal(st, st0)


def test_rng_state_roundtrip():
    r = gsct.Rng(77)
    for _ in range(500):
        r.uniform()
    s = r.state()
    a = [r.uniform() for _ in range(5)]
    r.set_state(s)
    assert [r.uniform() for _ in range(5)] == a


def _device_inputs(p, mom, acc):
    import torch
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    cloud = gsct.GaussianCloud(t(p["pos"]), t(p["ls"]), t(p["q"]), t(p["raw"]))
    n = cloud.size()
    st = gsct.OptimState(n, 0, 0)
    for k in KEYS:
        getattr(st, k).copy_(t(mom[k]))
    st.accum_grad_norm.copy_(t(acc["grad_norm"]))
    st.accum_grad_dir.copy_(t(acc["grad_dir"]))
    st.accum_count.copy_(t(acc["count"]))
    st.step, st.skipped_updates = 17, 3
    return cloud, st


@pytest.mark.gpu
@pytest.mark.parametrize("kind", CASES)
def test_adaptive_control_matches_reference(ref, ctx, kind):
    p, mom, acc, cfg, seed, pre = _case(kind)
    st_ref = _rng_state(seed, pre)
    op, om, rep = ref.adaptive_control(p, mom, acc, st_ref, **cfg)
    ops = _numpy_decisions(p, acc, cfg)

    cloud, st = _device_inputs(p, mom, acc)
    r = gsct.Rng(seed)
    for _ in range(pre):
        r.uniform()
    st.rng = r
    st.scene_extent = cfg["scene_extent"]
    conf = gsct.ControlConfig(cfg["grad_threshold"], cfg["prune_density"], cfg["split_scale_fraction"],
                              cfg["max_gaussians"])
    got = gsct.adaptive_control(cloud, st, conf, ctx=ctx)
    assert (got.pruned, got.cloned, got.split) == (rep["pruned"], rep["cloned"], rep["split"])
    m = rep["n_next"]
    assert cloud.size() == m
    st.check_lockstep(m)
    assert st.step == 17 and st.skipped_updates == 3
    s = st.rng.state()
    assert np.array_equal(np.array(list(s.x) + [s.p], dtype=np.uint64), st_ref), "engine state after the call"
    g = cloud.numpy()
    # which rows are fresh children (positions computed through log/cos) vs copies / nudges
    child = np.zeros(m, dtype=bool)
    nudged = np.zeros(m, dtype=bool)
    row = 0
    for o in ops:
        if o == 0:
            row += 1
        elif o == 2:
            nudged[row + 1] = True
            row += 2
        elif o == 3:
            child[row:row + 2] = True
            row += 2
    exact = ~(child | nudged)
    assert np.array_equal(g.positions[exact], op["pos"][exact])
    scale = np.abs(op["pos"]).max() + 1.0
    assert np.abs(g.positions[child] - op["pos"][child]).max(initial=0.0) <= 1e-12 * scale
    assert np.abs(g.positions[nudged] - op["pos"][nudged]).max(initial=0.0) <= 1e-13 * scale
    assert np.array_equal(g.log_scales, op["ls"])
    assert np.array_equal(g.rotations, op["q"])
    assert np.array_equal(g.raw_densities, op["raw"])
    for k in KEYS:
        assert np.array_equal(getattr(st, k).cpu().numpy(), om[k]), k
    assert not st.accum_grad_norm.any() and not st.accum_grad_dir.any() and not st.accum_count.any()


@pytest.mark.gpu
def test_accumulate_control_stats(ctx):
    import torch
    n = 1000
    rng = np.random.default_rng(4)
    g = gsct.ParamGradients.zeros(n, 0)
    g.positions.copy_(torch.from_numpy(rng.normal(size=(n, 3))))
    g.pos_grad_norm.copy_(torch.from_numpy(rng.uniform(size=n)))
    vis = (rng.random(n) < 0.6).astype(np.uint8)
    g.visible.copy_(torch.from_numpy(vis))
    st = gsct.OptimState(n, 0, 0)
    st.accum_grad_norm.fill_(0.5)
    st.accum_count.fill_(2)
    for _ in range(2):
        gsct.accumulate_control_stats(st, g, ctx=ctx)
    v = vis.astype(bool)
    want_norm = np.where(v, (0.5 + g.pos_grad_norm.cpu().numpy()) + g.pos_grad_norm.cpu().numpy(), 0.5)
    assert np.array_equal(st.accum_grad_norm.cpu().numpy(), want_norm)
    gp = g.positions.cpu().numpy()
    assert np.array_equal(st.accum_grad_dir.cpu().numpy(), np.where(v[:, None], gp + gp, 0.0))
    assert np.array_equal(st.accum_count.cpu().numpy(), np.where(v, 4, 2))


@pytest.mark.gpu
def test_adaptive_control_contract(ctx):
    import torch
    p, mom, acc, cfg, seed, pre = _case("calm")
    p["q"][9] = 0.0
    cloud, st = _device_inputs(p, mom, acc)
    with pytest.raises(gsct.ContractError, match="zero quaternion in splat 9"):
        gsct.adaptive_control(cloud, st, ctx=ctx)
    p, mom, acc, cfg, seed, pre = _case("calm")
    p["pos"][3, 1] = np.nan
    p["pos"][30, 1] = np.inf
    cloud, st = _device_inputs(p, mom, acc)
    with pytest.raises(gsct.ContractError, match="non-finite parameter in splat 3"):
        gsct.adaptive_control(cloud, st, ctx=ctx)
    cloud, st = _device_inputs(*_case("calm")[:3])
    st.accum_count = torch.zeros(5, dtype=torch.int64, device="cuda")
    with pytest.raises(gsct.ContractError, match="lockstep"):
        gsct.adaptive_control(cloud, st, ctx=ctx)


@pytest.mark.gpu
def test_adaptive_control_empty_and_all_pruned(ctx):
    import torch
    cloud, st = _device_inputs({"pos": np.zeros((0, 3)), "ls": np.zeros((0, 3)), "q": np.zeros((0, 4)),
                                "raw": np.zeros(0)},
                               {k: np.zeros((0, WIDTH[k]) if WIDTH[k] > 1 else (0,)) for k in KEYS},
                               {"grad_norm": np.zeros(0), "grad_dir": np.zeros((0, 3)),
                                "count": np.zeros(0, dtype=np.int64)})
    rep = gsct.adaptive_control(cloud, st, ctx=ctx)
    assert (rep.pruned, rep.cloned, rep.split) == (0, 0, 0) and cloud.size() == 0
    # every activated density zero: max density 0, prune_below 0, nothing is < 0 -> all kept
    p, mom, acc, cfg, seed, pre = _case("calm")
    p["raw"][:] = 0.0
    cloud, st = _device_inputs(p, mom, acc)
    rep = gsct.adaptive_control(cloud, st, ctx=ctx)
    assert rep.pruned == 0 and cloud.size() == len(p["raw"])
    assert torch.equal(cloud.positions.cpu(), torch.from_numpy(p["pos"]))
