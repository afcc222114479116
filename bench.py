#!/usr/bin/env python
"""bench.py — FaCT-GS hot paths on B200 (BASELINE.json metric).

Headline (`value`): fwd+bwd projections/s of the paper-standard workload (BASELINE.json
configs[1], SURVEY.md 8d "C2"): 75 cone-beam views at 512^2 of a 200k-Gaussian
Shepp-Logan phantom cloud in a 256^3 volume, one step = forward projection of all 75
views + backward (per-Gaussian gradients summed over the views), device-resident.
`e2e` is the same step through the C ABI with pinned HOST buffers (cloud up, grad images
up, images and gradients down inside the timed region). Secondary lines: fwd+bwd proj/s
at 2048^2 (1M Gaussians, C5) and voxelization Gvox/s at 512^3 (500k Gaussians, C3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (views sharded across ranks,
                                                         NCCL all-reduce of gradients)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fwd+bwd projections/s at 512² and 2k² vs CPU ref; voxelize Gvox/s at 512³"
UNIT = "projections/s"
WORKLOADS = {
    # name: (volume side, gaussians, views, detector side)
    "c1": (128, 50_000, 75, 256),
    "c2": (256, 200_000, 75, 512),
    "c4": (512, 400_000, 75, 1024),
    "c5": (1024, 1_000_000, 75, 2048),
}
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------------------
# workload construction (host, seeded; identical inputs for the GPU and the CPU reference)
# ---------------------------------------------------------------------------------------
def make_workload(name: str, seed: int = 0):
    from paper_2604_01844_b200 import gsct

    side, n, views, det = WORKLOADS[name]
    cloud = gsct.make_cloud("shepp_logan", n, seed=seed, side=side, spacing=1.0)
    geom = gsct.default_geometry((side, side, side), 1.0, views, "cone", det, det)
    return cloud, geom


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """View sharding: rank r owns views {v : v mod P == r}."""
    from paper_2604_01844_b200.sharding import shard_views as _sv

    return _sv(n_views, rank, world)


# ---------------------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9 and parts[1].isdigit():
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [int(r[1]) for r in rows]
        sm_max = max(int(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        loaded = [s for s in sm if s > 0.5 * sm_max] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": sm_max, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3] not in ("", "[N/A]"))}


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
class DeviceStep:
    """One fwd+bwd pass over this rank's views with device-resident inputs/outputs."""

    def __init__(self, ctx, cloud, geom, views, world: int):
        import torch
        from paper_2604_01844_b200 import gsct

        self.gsct, self.torch, self.ctx = gsct, torch, ctx
        self.geom, self.views, self.world = geom, views, world
        self.dev = torch.device(f"cuda:{ctx.device}")
        self.dcloud = cloud.to_device(ctx.device)
        n = cloud.size()
        nv = len(views)
        self.images = torch.empty((nv, geom.n_v, geom.n_u), dtype=torch.float32, device=self.dev)
        # dL/dimage: all-ones, as the reference sweep (bench.hpp:114-115)
        self.grad_images = torch.ones((nv, geom.n_v, geom.n_u), dtype=torch.float32, device=self.dev)
        # one flat fp64 buffer so a single all-reduce carries every gradient class
        from paper_2604_01844_b200.sharding import pack_grads

        self.flat, self.grads = pack_grads(n, like=self.images)
        self.stream = torch.cuda.ExternalStream(int(gsct.lib().gsct_ctx_stream(ctx.handle)), device=self.dev)
        self.rs = gsct.RasterSettings()
        # training-loop usage: the backward reuses the forward's set-up (same cloud)
        ctx.set_save_for_backward(True)

    def __call__(self):
        g = self.gsct
        g.rasterize_views(self.dcloud, self.geom, self.views, self.rs, out=self.images, ctx=self.ctx)
        g.rasterize_backward_views(self.dcloud, self.geom, self.views, self.grad_images, self.rs, out=self.grads,
                                   ctx=self.ctx)
        if self.world > 1:
            from paper_2604_01844_b200.sharding import allreduce_grads

            with self.torch.cuda.stream(self.stream):  # NCCL on the library's stream, no host sync
                allreduce_grads(self.flat, self.grads.visible)


def timed_steps(step, stream, k: int, flush) -> list[float]:
    import torch

    times = []
    for _ in range(k):
        with torch.cuda.stream(stream):
            flush()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    return times


def run_e2e(ctx, cloud, geom, views, k: int, w: int, world: int = 1) -> dict:
    """Same step through the C ABI with pinned host buffers; copies inside the timed region.
    With several ranks each rank runs its view shard and the summed gradients are formed by
    an all-reduce of the packed fp64 gradient buffer (host -> device -> all-reduce -> host,
    inside the step); per-step time = max over ranks."""
    import torch
    from paper_2604_01844_b200 import gsct

    ctx.set_async(False)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    hcloud = gsct.GaussianCloud(pin(cloud.positions), pin(cloud.log_scales), pin(cloud.rotations),
                                pin(cloud.raw_densities))
    nv = len(views)
    n = cloud.size()
    images = torch.empty((nv, geom.n_v, geom.n_u), dtype=torch.float32).pin_memory().numpy()
    gimg = torch.ones((nv, geom.n_v, geom.n_u), dtype=torch.float32).pin_memory().numpy()
    # one pinned fp64 buffer holding every gradient class (pos 3N, ls 3N, q 4N, raw N, |g2d| N)
    flat_h = torch.zeros(12 * n, dtype=torch.float64).pin_memory()
    f = flat_h.numpy()
    grads = gsct.ParamGradients(f[:3 * n].reshape(n, 3), f[3 * n:6 * n].reshape(n, 3), f[6 * n:10 * n].reshape(n, 4),
                                f[10 * n:11 * n], f[11 * n:], torch.zeros(n, dtype=torch.uint8).pin_memory().numpy())
    rs = gsct.RasterSettings()
    dev = torch.device(f"cuda:{ctx.device}")
    flat_d = torch.empty(12 * n, dtype=torch.float64, device=dev) if world > 1 else None

    def step():
        gsct.rasterize_views(hcloud, geom, views, rs, out=images, ctx=ctx)
        gsct.rasterize_backward_views(hcloud, geom, views, gimg, rs, out=grads, ctx=ctx)
        if world > 1:
            import torch.distributed as dist

            flat_d.copy_(flat_h, non_blocking=True)
            dist.all_reduce(flat_d)
            flat_h.copy_(flat_d)  # device->host: the summed gradients
        return float(grads.raw_densities[0])  # device->host result read

    for _ in range(w):
        step()
    ts = []
    for _ in range(k):
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        t0 = time.perf_counter()
        step()
        ts.append((time.perf_counter() - t0) * 1e3)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor(ts, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ts = t.cpu().tolist()
    cloud_bytes = n * 11 * 8
    h2d = 2 * cloud_bytes + gimg.nbytes + (flat_h.numel() * 8 if world > 1 else 0)  # cloud up in both calls
    d2h = images.nbytes + n * (12 * 8 + 1) + (flat_h.numel() * 8 if world > 1 else 0)
    return {"ms": ts, "h2d": h2d, "d2h": d2h}


def cpu_baseline_sample(cloud, geom, budget_s: float = 10.0, max_views: int = 75) -> dict:
    """The unchanged reference (oracle/_ref/libgsct_ref.so) on every host core: fwd+bwd of
    the first views of the same workload until the time budget (bounded sample)."""
    from oracle.oracle import Ref
    from paper_2604_01844_b200 import gsct

    ref = Ref()
    cores = ref.threads()
    h = ref.cloud(cloud)
    rs = gsct.RasterSettings()
    ones = np.ones((geom.n_v, geom.n_u))
    n = cloud.size()
    done, t_total = 0, 0.0
    try:
        while done < max_views and t_total < budget_s:
            t0 = time.perf_counter()
            ref.rasterize_view(h, geom, done, rs)
            ref.rasterize_backward(h, geom, done, ones, rs, n)
            t_total += time.perf_counter() - t0
            done += 1
    finally:
        ref.free_cloud(h)
    return {"value": done / t_total, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"first {done} of {len(geom.angles)} views, fwd+bwd (rasterize_view + rasterize_backward), "
                      f"{t_total:.1f} s wall on {cores} threads; per-view rate"}


def secondary_2k(ctx, n_views_measured: int = 8, k: int = 3) -> dict:
    import torch
    from paper_2604_01844_b200 import gsct

    cloud, geom = make_workload("c5")
    views = list(range(n_views_measured))
    st = DeviceStep(ctx, cloud, geom, views, 1)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=st.dev)
    st()
    ts = timed_steps(st, st.stream, k, lambda: flush.zero_())
    ms = float(np.mean(ts))
    return {"proj_per_s_2048": n_views_measured / (ms / 1e3), "workload": "C5: 1M Gaussians, 1024^3 SL cloud, "
            f"cone 2048^2, fwd+bwd of {n_views_measured} of 75 views per step (per-view rate)", "ms_per_step": ms}


def secondary_train(ctx, k: int = 5) -> dict:
    """BASELINE configs[1] as a device-resident training iteration: render the 75 C2 views,
    fused L1 + 0.25 SSIM2D image loss against measured projections (rendered from the
    unperturbed cloud), backward to the Gaussians, one Adam step (batched-gradient data
    parallelism: one optimiser step per 75-view batch)."""
    import torch
    from paper_2604_01844_b200 import gsct

    cloud, geom = make_workload("c2")
    dev = torch.device(f"cuda:{ctx.device}")
    views = list(range(len(geom.angles)))
    target = cloud.to_device(ctx.device)
    measured = gsct.rasterize_views(target, geom, views, gsct.RasterSettings(), ctx=ctx)
    rng = np.random.default_rng(3)
    pert = gsct.GaussianCloud(cloud.positions + rng.normal(0, 0.3, cloud.positions.shape), cloud.log_scales,
                              cloud.rotations, cloud.raw_densities * 0.9)
    st = DeviceStep(ctx, pert, geom, views, 1)
    adam = gsct.AdamState(pert.size(), ctx.device)
    lrs = gsct.LearningRates()
    losses = []

    def it():
        gsct.rasterize_views(st.dcloud, geom, views, st.rs, out=st.images, ctx=ctx)
        lv, _ = gsct.image_loss(st.images, measured, 0.25, grad_out=st.grad_images, ctx=ctx)
        gsct.rasterize_backward_views(st.dcloud, geom, views, st.grad_images, st.rs, out=st.grads, ctx=ctx)
        gsct.adam_step(st.dcloud, adam, st.grads, lrs, ctx=ctx)
        losses.append(float(lv[:, 2].mean()))

    it()
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    ts = timed_steps(it, st.stream, k, lambda: flush.zero_())
    ms = float(np.mean(ts))
    return {"workload": "C2 training iteration: 75 views render + L1/SSIM2D loss + backward + Adam (device-resident)",
            "ms_per_iteration": ms, "proj_per_s": len(views) / (ms / 1e3),
            "mean_view_loss_first_last": [losses[0], losses[-1]], "iterations": len(losses)}


def secondary_voxel(ctx, k: int = 3) -> dict:
    import torch
    from paper_2604_01844_b200 import gsct

    side, n = 512, 500_000
    cloud = gsct.make_cloud("shepp_logan", n, seed=1, side=side, spacing=1.0).to_device(ctx.device)
    grid = gsct.GridSpec.centered((side, side, side), 1.0)
    region = gsct.GridRegion.covering(grid)
    vs = gsct.VoxelSettings()
    dev = torch.device(f"cuda:{ctx.device}")
    vol = torch.empty((side, side, side), dtype=torch.float32, device=dev)
    gvol = torch.ones_like(vol)
    grads = gsct.ParamGradients.zeros(n, ctx.device)
    stream = torch.cuda.ExternalStream(int(gsct.lib().gsct_ctx_stream(ctx.handle)), device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    fwd = lambda: gsct.voxelize(cloud, region, vs, out=vol, ctx=ctx)
    bwd = lambda: gsct.voxelize_backward(cloud, region, gvol, vs, out=grads, ctx=ctx)
    stats = gsct.RenderStats()
    ctx.set_async(False)
    gsct.voxelize(cloud, region, vs, stats, out=vol, ctx=ctx)
    ctx.set_async(True)
    fwd()
    bwd()
    tf = float(np.mean(timed_steps(fwd, stream, k, lambda: flush.zero_())))
    tb = float(np.mean(timed_steps(bwd, stream, k, lambda: flush.zero_())))
    nvox = side ** 3
    return {"voxelize_gvox_per_s_512": nvox / (tf / 1e3) / 1e9, "voxelize_fwd_bwd_gvox_per_s_512":
            nvox / ((tf + tb) / 1e3) / 1e9, "fwd_ms": tf, "bwd_ms": tb, "voxel_pairs": stats.pixel_pairs,
            "workload": "C3: 500k Gaussians (SL cloud), 512^3 grid, voxelize_full + voxelize_backward"}


def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_2604_01844_b200 import gsct

    torch.cuda.set_device(local_rank)
    ctx = gsct.context(local_rank)
    cloud, geom = make_workload(args.config)
    views = shard_views(len(geom.angles), rank, world)
    step = DeviceStep(ctx, cloud, geom, views, world)
    flush_buf = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=step.dev)

    # exact work counters of one step (RenderStats), untimed
    ctx.set_async(False)
    stats = gsct.RenderStats()
    gsct.rasterize_views(step.dcloud, geom, views, step.rs, stats, out=step.images, ctx=ctx)
    ctx.set_async(True)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = ctx.launch_count()
    ctx.set_profiling(True)
    ctx.phase_times()
    with ClockSampler(local_rank) as clk:
        ts = timed_steps(step, step.stream, args.steps, lambda: flush_buf.zero_())
    phases = ctx.phase_times()
    ctx.set_profiling(False)
    launches = ctx.launch_count() - launches0
    torch.cuda.synchronize()
    total_ms = float(np.sum(ts))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=step.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    n_views_total = len(geom.angles)
    value = n_views_total * args.steps / (total_ms / 1e3)

    # e2e through the C ABI with pinned host buffers (every rank: its shard + the all-reduce)
    e2e = None
    if not args.no_e2e:
        e = run_e2e(ctx, cloud, geom, views, max(3, min(args.steps, 5)), 2, world)
        e_ms = float(np.mean(e["ms"]))
        e2e = {"value": round(n_views_total / (e_ms / 1e3), 2), "unit": UNIT, "h2d_bytes_per_step": e["h2d"],
               "d2h_bytes_per_step": e["d2h"], "ms_per_step": round(e_ms, 3),
               "path": "gsct_rasterize_fwd + gsct_rasterize_bwd (C ABI, GSCT_HOST pinned buffers, sync)"
                       + (" + all-reduce of the packed gradients, max over ranks" if world > 1 else "")}
        ctx.set_async(True)

    if rank != 0:
        return

    # --- roofline of the dominant kernel (live CUDA-event phase timing over the timed region)
    ex2_peak = ctx.microbench("ex2")
    ffma_peak = ctx.microbench("ffma")
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    dom = max(("raster_fwd", "raster_bwd"), key=lambda p: phases[p][0])
    dom_ms, dom_count = phases[dom]
    launches_per_step = max(dom_count // args.steps, 1)  # views are processed in chunks
    avg_ms = dom_ms / max(dom_count, 1)
    n = cloud.size()
    nv = len(views)
    npx = geom.n_u * geom.n_v
    # compulsory bytes per step: the 32 B fp32 splat record of every
    # (view, splat) read once + the image write (fwd) / the grad-image read and the 32 B
    # moment write (bwd); per launch = per step / launches (equal-size view chunks)
    items = nv * n
    algo_bytes_step = items * 32 + nv * npx * 4 + (items * 32 if dom == "raster_bwd" else 0)
    algo_bytes = algo_bytes_step / launches_per_step
    pairs_per_launch = stats.pixel_pairs / launches_per_step
    achieved_gbs = algo_bytes / (avg_ms / 1e3) / 1e9
    pair_rate = pairs_per_launch / (avg_ms / 1e3)
    kernel = "k_raster_fwd4" if dom == "raster_fwd" else "k_raster_bwd_lanes"
    traffic = None  # dram read+write bytes per launch from the committed ncu --set full capture
    measured = None  # the pipes that do bind (same capture): issue slots, L1/L2 throughput
    try:
        prof = json.loads((ROOT / "profiles" / "r1" / "raster" / "summary.json").read_text())
        hit = [d for d in prof if d["kernel"] == kernel and "dram_bytes" in d]
        if hit and args.config == "c2":
            traffic = int(np.mean([d["dram_bytes"] for d in hit]))
            measured = {"kernel": kernel, "source": "profiles/r1/raster/summary.json (ncu --set full, C2)"}
            for key in ("issue_active_pct", "l1tex_throughput_pct", "l1_lsu_wavefronts_pct", "l2_throughput_pct", "xu_pipe_pct",
                        "fma_pipe_pct", "warps_active_pct"):
                if key in hit[0]:
                    measured[key] = round(float(np.mean([d[key] for d in hit])), 1)
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": kernel,
                "achieved": round(achieved_gbs, 2), "peak": hbm_peak,
                "unit": "GB/s", "frac": round(achieved_gbs / hbm_peak, 4), "traffic": traffic,
                "peak_source": hbm_src, "algorithmic_bytes_per_launch": int(algo_bytes),
                "avg_launch_ms": round(avg_ms, 4), "launches_per_step": launches_per_step,
                "note": "not HBM-bound by design: the binding resources are SFU/issue (roofline_sfu)"}
    roofline_sfu = {"bound": "sfu_ex2", "kernel": roofline["kernel"], "achieved": pair_rate, "peak": ex2_peak,
                    "unit": "ex2/s (= splat-pixel pairs/s)", "frac": round(pair_rate / ex2_peak, 4),
                    "pairs_per_launch": int(pairs_per_launch), "ffma_peak_per_s": ffma_peak,
                    "note": "one exp per splat-pixel pair per pass (projector.hpp:341,410); peak = on-box "
                            "MUFU ex2.approx microbenchmark in this run"}

    out = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded 3D Shepp-Logan phantom cloud, random init)",
        "config": {"workload": f"{args.config.upper()}: {n} Gaussians, {WORKLOADS[args.config][0]}^3 volume, "
                               f"{n_views_total} cone views at {geom.n_u}^2, fwd+bwd per step",
                   "gaussians": n, "views": n_views_total, "detector": [geom.n_u, geom.n_v],
                   "volume_side": WORKLOADS[args.config][0], "parallelism": f"views sharded over {world} GPU(s)",
                   "l2": "flushed between timed steps (256 MiB memset outside the events)",
                   "settings": "reference defaults: tau 1e-4, sigma_cap 3, 16x16 tiles, 0.3 px^2 dilation"},
        "work": {"tile_pairs_per_step": stats.tile_pairs, "pixel_pairs_per_pass": stats.pixel_pairs,
                 "culled": stats.culled, "degenerate": stats.degenerate},
        "roofline": roofline, "roofline_sfu": roofline_sfu, "roofline_measured": measured,
        "phase_ms_per_step": {k: round(v[0] / args.steps, 4) for k, v in phases.items() if v[1]},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    if e2e is not None:
        out["e2e"] = e2e
    if not args.no_secondary and world == 1:
        try:
            out["secondary"] = {"raster_2048": secondary_2k(ctx), "voxel_512": secondary_voxel(ctx),
                                "train_iteration_c2": secondary_train(ctx)}
        except Exception as exc:  # report, never hide the main line
            out["secondary"] = {"error": repr(exc)}
    if not args.no_cpu_baseline and world == 1:
        try:
            out["cpu_baseline"] = cpu_baseline_sample(cloud, geom)
        except Exception as exc:
            out["cpu_baseline"] = {"error": repr(exc)}
    print(json.dumps(out), flush=True)


def run_reference(args, rank: int, world: int) -> None:
    """Reference arm: the reference's own CPU implementation (oracle/_ref, compiled from the
    unchanged /root/reference headers) on all host threads, same metric and workload."""
    if rank != 0:
        return
    from oracle.oracle import REF_LIB, Ref
    from paper_2604_01844_b200 import gsct

    if not REF_LIB.exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libgsct_ref.so was not built"}))
        return
    cloud, geom = make_workload(args.config)
    ref = Ref()
    cores = ref.threads()
    h = ref.cloud(cloud)
    rs = gsct.RasterSettings()
    ones = np.ones((geom.n_v, geom.n_u))
    n = cloud.size()
    views_per_step = 1

    def step(i):
        v = i % len(geom.angles)
        ref.rasterize_view(h, geom, v, rs)
        ref.rasterize_backward(h, geom, v, ones, rs, n)

    for i in range(args.warmup):
        step(i)
    ts = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        step(args.warmup + i)
        ts.append((time.perf_counter() - t0) * 1e3)
    ref.free_cloud(h)
    ms = float(np.mean(ts))
    value = views_per_step / (ms / 1e3)
    sample = (f"{views_per_step} of {len(geom.angles)} views fwd+bwd per step (rasterize_view + "
              f"rasterize_backward), {cores} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded 3D Shepp-Logan cloud)",
        "config": {"workload": f"{args.config.upper()}: {n} Gaussians, {len(geom.angles)} cone views at "
                               f"{geom.n_u}^2, fwd+bwd (bounded per-step sample)"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # plumbing check only: gloo lets several ranks share one GPU (NCCL refuses duplicate
    # devices); the real multi-GPU run uses the default nccl
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        log("note: the timing rules require >= 3 warm-up steps")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours" and world > 1 and args.dist_backend == "gloo":
        import torch

        local_rank %= max(torch.cuda.device_count(), 1)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
        else:
            dist.init_process_group("gloo")
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
