#!/usr/bin/env python
"""bench.py — FaCT-GS hot paths on B200 (BASELINE.json metric).

Headline (`value`): fwd+bwd projections/s of the paper-standard workload (BASELINE.json
configs[1], SURVEY.md 8d "C2"): 75 cone-beam views at 512^2 of a 200k-Gaussian
Shepp-Logan phantom cloud in a 256^3 volume, one step = forward projection of all 75
views + backward (per-Gaussian gradients summed over the views), device-resident.
`e2e` is the same step through the C ABI with pinned HOST buffers (cloud up, grad images
up, images and gradients down inside the timed region). The other two metric numbers are
full lines of their own under `secondary`: fwd+bwd proj/s at 2048^2 (C5: 1M Gaussians, all
75 views per step) and voxelization Gvox/s at 512^3 (C3: 500k Gaussians) plus 1024^3 (C5's
volume), each with a roofline object and the reference CPU figure.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (views sharded across ranks,
                                                         NCCL all-reduce of gradients)
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
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
# SURVEY.md 8(d) compulsory bytes: per splat 44 B of parameters read per pass, 49 B of
# gradients written by the backward; 4 B per pixel / voxel written (forward) or read (backward)
PARAM_B, GRAD_B, PX_B = 44, 49, 4
# FMA-pipe ops per pair the reference formulation costs: fwd ~4, raster bwd
# ~12, voxel bwd ~20 (the FMA sub-bound beside the MUFU-pair bound)
FMA_PER_PAIR = {"raster_fwd": 4, "raster_bwd": 12, "voxel_fwd": 4, "voxel_bwd": 20}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_for(name: str, world: int = 1) -> dict:
    """The workload description shared by both arms (same string, same keys)."""
    side, n, views, det = WORKLOADS[name]
    return {"workload": f"{name.upper()}: {n} Gaussians (seeded 3D Shepp-Logan phantom cloud), {side}^3 volume, "
                        f"{views} cone views at {det}^2, fwd+bwd of every view per step",
            "gaussians": n, "views": views, "detector": [det, det], "volume_side": side,
            "parallelism": f"views sharded over {world} GPU(s)",
            "l2": "flushed between timed steps (256 MiB memset outside the events)",
            "settings": "reference defaults: tau 1e-4, sigma_cap 3, 16x16 tiles, 0.3 px^2 dilation",
            "grad_images": "all-ones (bench.hpp:114-115)"}


# ---------------------------------------------------------------------------------------
# workload construction (host, seeded; identical inputs for the GPU and the CPU reference)
# ---------------------------------------------------------------------------------------
def make_workload(name: str, seed: int = 0):
    from paper_2604_01844_b200 import gsct

    side, n, views, det = WORKLOADS[name]
    cloud = gsct.make_cloud("shepp_logan", n, seed=seed, side=side, spacing=1.0)
    geom = gsct.default_geometry((side, side, side), 1.0, views, "cone", det, det)
    return cloud, geom


def make_workload_ref(ref, name: str, seed: int = 0):
    """The same inputs built without the product library: the phantom cloud drawn with the
    reference's Rng and default_geometry (synthetic.hpp:246-271) from oracle/_ref
    (bit-identical to make_workload: tests/test_capi.py)."""
    from paper_2604_01844_b200.gsct import GaussianCloud, ScanGeometry  # pure-Python value types

    side, n, views, det = WORKLOADS[name]
    pos, ls, q, raw = ref.shepp_logan_cloud(n, side, 1.0, seed)
    g, ang = ref.default_geometry((side, side, side), 1.0, views, 1, det, det)
    geom = ScanGeometry("cone", g.n_u, g.n_v, g.s_u, g.s_v, list(ang), g.source_to_origin, g.origin_to_detector)
    return GaussianCloud(pos, ls, q, raw), geom


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """View sharding: rank r owns views {v : v mod P == r}."""
    from paper_2604_01844_b200.sharding import shard_views as _sv

    return _sv(n_views, rank, world)


# ---------------------------------------------------------------------------------------
# clocks sampled DURING the timed region (NVML in a thread, 2 ms period)
# ---------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int, period_s: float = 0.002):
        self.device, self.period = device, period_s
        self.rows: list[tuple[int, int, int, float]] = []  # (sm MHz, max MHz, reasons, power W)
        self._stop = threading.Event()
        self._thr = None
        self._nv = None

    def _sample(self):
        nv, h = self._nv, self._h
        try:
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
            self.rows.append((int(sm), int(self._smax), int(rs), float(pw)))
        except Exception:
            pass

    def _poll(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self._nv, self._h = nv, nv.nvmlDeviceGetHandleByIndex(self.device)
            self._smax = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._sample()  # at the start of the timed region (the GPU is busy with the warm-up)
            self._switch = sys.getswitchinterval()
            sys.setswitchinterval(0.0005)  # let the sampling thread in between launches
            self._thr = threading.Thread(target=self._poll, daemon=True)
            self._thr.start()
            time.sleep(0.01)
        except Exception:
            self._nv = None
        return self

    def __exit__(self, *exc):
        if self._nv is not None:
            self._sample()  # the end of the timed region
            sys.setswitchinterval(self._switch)
        self._stop.set()
        if self._thr is not None:
            self._thr.join(timeout=2)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        sm_max = max(r[1] for r in self.rows)
        reasons = sorted({name for r in self.rows for bit, name in self.REASONS.items() if r[2] & bit})
        loaded = [s for s in sm if s > 0.5 * sm_max] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": sm_max, "reasons": reasons,
                "samples": len(self.rows), "power_w_max": round(max(r[3] for r in self.rows), 1),
                "source": "NVML, 2 ms period, inside the timed region"}


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
class DeviceStep:
    """One fwd+bwd pass over this rank's views with device-resident inputs/outputs."""

    def __init__(self, ctx, cloud, geom, views, world: int, native_group: bool = False):
        import torch
        from paper_2604_01844_b200 import gsct

        self.gsct, self.torch, self.ctx = gsct, torch, ctx
        self.geom, self.views, self.world = geom, views, world
        # native_group: the context carries the library's NCCL group, so gsct_rasterize_bwd
        # itself all-reduces the per-splat view sums on its stream (include/gsct_cuda.h)
        self.native_group = native_group
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
        if self.world > 1 and not self.native_group:
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


def run_e2e(ctx, cloud, geom, views, k: int, w: int, world: int = 1, native_group: bool = False) -> dict:
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
    torch_reduce = world > 1 and not native_group  # with the native group the call reduces itself
    flat_d = torch.empty(12 * n, dtype=torch.float64, device=dev) if torch_reduce else None

    def step():
        gsct.rasterize_views(hcloud, geom, views, rs, out=images, ctx=ctx)
        gsct.rasterize_backward_views(hcloud, geom, views, gimg, rs, out=grads, ctx=ctx)
        if torch_reduce:
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
    h2d = 2 * cloud_bytes + gimg.nbytes + (flat_h.numel() * 8 if torch_reduce else 0)  # cloud up in both calls
    d2h = images.nbytes + n * (12 * 8 + 1) + (flat_h.numel() * 8 if torch_reduce else 0)
    return {"ms": ts, "h2d": h2d, "d2h": d2h}


# ---------------------------------------------------------------------------------------
# roofline objects (live CUDA-event kernel phases; SURVEY.md 8d units)
# ---------------------------------------------------------------------------------------
def _peaks(ctx) -> dict:
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    return {"hbm": peaks.get("hbm_gbs", 6650.0),
            "hbm_src": "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)",
            "ex2": ctx.microbench("ex2"), "ffma": ctx.microbench("ffma")}


def _ncu_traffic(tag: str, kernel: str):
    """dram read+write bytes per launch of `kernel` from the committed ncu --set full summary."""
    try:
        prof = json.loads((ROOT / "profiles" / tag / "summary.json").read_text())
        hit = [d for d in prof if d["kernel"] == kernel and "dram_bytes" in d]
        if hit:
            return int(np.mean([d["dram_bytes"] for d in hit])), hit[0]
    except Exception:
        pass
    return None, None


def roofline_objects(peaks: dict, phase: str, kernel: str, ms_total: float, launches: int, algo_bytes_step: float,
                     pairs_step: float, steps: int, ncu_tag: str) -> tuple[dict, dict]:
    """`roofline` (HBM: SURVEY 8d compulsory bytes of the kernel's launches / its measured
    launch time) and `roofline_sfu` (splat-pair rate vs the on-box MUFU ex2 peak, the bound
    SURVEY 8d names; the FMA sub-bound beside it)."""
    launches_per_step = max(launches // max(steps, 1), 1)
    avg_ms = ms_total / max(launches, 1)
    algo_bytes = algo_bytes_step / launches_per_step
    pairs = pairs_step / launches_per_step
    achieved = algo_bytes / (avg_ms / 1e3) / 1e9
    rate = pairs / (avg_ms / 1e3)
    traffic, meas = _ncu_traffic(ncu_tag, kernel)
    roof = {"bound": "hbm", "kernel": kernel, "achieved": round(achieved, 2), "peak": peaks["hbm"], "unit": "GB/s",
            "frac": round(achieved / peaks["hbm"], 4), "traffic": traffic, "peak_source": peaks["hbm_src"],
            "algorithmic_bytes_per_launch": int(algo_bytes), "avg_launch_ms": round(avg_ms, 4),
            "launches_per_step": launches_per_step,
            "algorithmic_bytes_def": "SURVEY.md 8(d): 44 B params read + 49 B grads written (bwd) per (view, splat), "
                                     "4 B per pixel/voxel written (fwd) or read (bwd)",
            "note": "compulsory HBM bytes are a few % of peak by design (neither path is bandwidth-bound); "
                    "the binding unit is named in 'binding' from the committed ncu capture, the pair rate "
                    "against the on-box MUFU / FFMA peaks is in roofline_sfu"}
    if meas:
        roof["ncu"] = {k: meas[k] for k in ("issue_active_pct", "fma_pipe_pct", "xu_pipe_pct", "l1tex_throughput_pct",
                                             "warps_active_pct", "duration_ms") if k in meas}
        roof["ncu"]["source"] = f"profiles/{ncu_tag}/summary.json"
        util = {"L1TEX (data pipe / wavefronts)": meas.get("l1tex_throughput_pct"),
                "FMA pipe": meas.get("fma_pipe_pct"), "issue": meas.get("issue_active_pct"),
                "XU (MUFU)": meas.get("xu_pipe_pct")}
        util = {k: v for k, v in util.items() if v is not None}
        if util:
            top = max(util, key=util.get)
            roof["binding"] = {"unit": top, "pct_of_peak": round(util[top], 1), "source": roof["ncu"]["source"]}
    fma = FMA_PER_PAIR[phase]
    sfu = {"bound": "sfu_ex2", "kernel": kernel, "achieved": rate, "peak": peaks["ex2"],
           "unit": "splat-pairs/s (one exp per pair in the reference, projector.hpp:341,410 / voxelizer.hpp:184,242)",
           "frac": round(rate / peaks["ex2"], 4), "pairs_per_launch": int(pairs),
           "fma_subbound": {"ops_per_pair": fma, "peak_ffma_per_s": peaks["ffma"],
                            "frac": round(rate * fma / peaks["ffma"], 4)},
           "note": "peaks = on-box MUFU ex2.approx / FFMA microbenchmarks in this run"}
    return roof, sfu


def cpu_baseline_views(ref, cloud, geom, n_views: int, budget_s: float = 15.0) -> dict:
    """The unchanged reference on every host core: fwd+bwd of the first views (bounded)."""
    from paper_2604_01844_b200.gsct import RasterSettings

    cores = ref.threads()
    h = ref.cloud(cloud)
    rs = RasterSettings()
    ones = np.ones((geom.n_v, geom.n_u))
    n = cloud.size()
    done, t_total = 0, 0.0
    try:
        while done < n_views and t_total < budget_s:
            t0 = time.perf_counter()
            ref.rasterize_view(h, geom, done, rs)
            ref.rasterize_backward(h, geom, done, ones, rs, n)
            t_total += time.perf_counter() - t0
            done += 1
    finally:
        ref.free_cloud(h)
    return {"value": round(done / t_total, 4), "unit": UNIT, "cores": cores, "kind": "reference",
            "cpu": cpu_model(),
            "sample": f"first {done} of {len(geom.angles)} views, fwd+bwd (rasterize_view + rasterize_backward, "
                      f"projector.hpp:308,371), {t_total:.1f} s wall on {cores} threads; per-view rate"
                      + (" (75-view step extrapolated linearly)" if done < len(geom.angles) else "")}


def cpu_baseline_voxel(ref, cloud, side: int, slices: int = 64, with_bwd: bool = True) -> dict:
    """The reference's voxelize (+ voxelize_backward) on a z-slab of `slices` slices of the
    side^3 grid (GridRegion::of_parent, voxelizer.hpp:53-66), all host threads; Gvox/s of the
    slab extrapolated to the full grid (labelled)."""
    from paper_2604_01844_b200.gsct import GridRegion, GridSpec, VoxelSettings

    cores = ref.threads()
    grid = GridSpec.centered((side,) * 3, 1.0)
    z0 = side // 2 - slices // 2
    region = GridRegion.of_parent(grid, (0, 0, z0), (side, side, slices))
    vs = VoxelSettings()
    h = ref.cloud(cloud)
    try:
        t0 = time.perf_counter()
        vol, _ = ref.voxelize(h, region, vs)
        tf = time.perf_counter() - t0
        tb = 0.0
        if with_bwd:
            gv = np.ones_like(vol)
            t0 = time.perf_counter()
            ref.voxelize_backward(h, region, gv, vs, cloud.size())
            tb = time.perf_counter() - t0
    finally:
        ref.free_cloud(h)
    nvox = side * side * slices
    out = {"value": round(nvox / (tf + tb) / 1e9, 6), "unit": "Gvox/s", "cores": cores, "kind": "reference",
           "cpu": cpu_model(), "fwd_gvox_per_s": round(nvox / tf / 1e9, 6),
           "sample": f"{slices}-slice z-slab ({side}x{side}x{slices}) of the {side}^3 grid, voxelize"
                     + (" + voxelize_backward (ones)" if with_bwd else "") +
                     f" (voxelizer.hpp:162,214), {tf + tb:.1f} s wall on {cores} threads; Gvox/s extrapolated to "
                     f"the full grid"}
    return out


# ---------------------------------------------------------------------------------------
# secondary lines: C5 (2048^2, 75 views), C3 (512^3), C5 volume (1024^3), C2 training step
# ---------------------------------------------------------------------------------------
def secondary_2k(ctx, peaks, ref, k: int = 5) -> dict:
    import torch

    cloud, geom = make_workload("c5")
    views = list(range(len(geom.angles)))
    st = DeviceStep(ctx, cloud, geom, views, 1)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=st.dev)
    from paper_2604_01844_b200 import gsct

    stats = gsct.RenderStats()
    ctx.set_async(False)
    gsct.rasterize_views(st.dcloud, geom, views, st.rs, stats, out=st.images, ctx=ctx)
    ctx.set_async(True)
    for _ in range(3):
        st()
    ctx.set_profiling(True)
    ctx.phase_times()
    ts = timed_steps(st, st.stream, k, lambda: flush.zero_())
    ph = ctx.phase_times()
    ctx.set_profiling(False)
    ms = float(np.mean(ts))
    n, nv, npx = cloud.size(), len(views), geom.n_u * geom.n_v
    dom = max(("raster_fwd", "raster_bwd"), key=lambda p: ph[p][0])
    bytes_step = nv * ((PARAM_B + (GRAD_B if dom == "raster_bwd" else 0)) * n + PX_B * npx)
    roof, sfu = roofline_objects(peaks, dom, "k_raster_fwd4" if dom == "raster_fwd" else "k_raster_bwd_chain",
                                 ph[dom][0], ph[dom][1], bytes_step, stats.pixel_pairs, k, "r2/raster_c5")
    out = {"metric": "fwd+bwd projections/s at 2048^2", "value": round(nv / (ms / 1e3), 2), "unit": UNIT,
           "ms_per_step": round(ms, 3), "steps": k, "warmup": 3, "step_ms": [round(t, 2) for t in ts],
           "config": {"workload": "C5: 1M Gaussians (3D Shepp-Logan phantom cloud), 1024^3 volume, 75 cone views "
                                  "at 2048^2, fwd+bwd of every view per step (device-resident, L2 flushed)"},
           "work": {"pixel_pairs_per_pass": stats.pixel_pairs, "tile_pairs_per_step": stats.tile_pairs},
           "phase_ms_per_step": {p: round(v[0] / k, 3) for p, v in ph.items() if v[1]},
           "roofline": roof, "roofline_sfu": sfu}
    if ref is not None:
        out["cpu_baseline"] = cpu_baseline_views(ref, cloud, geom, 3, budget_s=60.0)
    del st
    torch.cuda.empty_cache()
    return out


def _voxel_line(ctx, peaks, ref, side: int, n: int, seed: int, k: int, ncu_tag: str, name: str) -> dict:
    import torch
    from paper_2604_01844_b200 import gsct

    cloud_h = gsct.make_cloud("shepp_logan", n, seed=seed, side=side, spacing=1.0)
    cloud = cloud_h.to_device(ctx.device)
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
    for _ in range(3):
        fwd()
        bwd()
    ctx.set_profiling(True)
    ctx.phase_times()
    tf = float(np.mean(timed_steps(fwd, stream, k, lambda: flush.zero_())))
    phf = ctx.phase_times()
    tb = float(np.mean(timed_steps(bwd, stream, k, lambda: flush.zero_())))
    phb = ctx.phase_times()
    ctx.set_profiling(False)
    nvox = side ** 3
    # dominant kernel of the fwd+bwd pair
    f_ms, f_cnt = phf["voxel_fwd"]
    b_ms, b_cnt = phb["voxel_bwd"]
    if b_ms >= f_ms:
        roof, sfu = roofline_objects(peaks, "voxel_bwd", "k_voxel_bwd_lanes", b_ms, b_cnt,
                                     PX_B * nvox + (PARAM_B + GRAD_B) * n, stats.pixel_pairs, k, ncu_tag)
    else:
        roof, sfu = roofline_objects(peaks, "voxel_fwd", "k_voxel_fwd2", f_ms, f_cnt, PX_B * nvox + PARAM_B * n,
                                     stats.pixel_pairs, k, ncu_tag)
    out = {"metric": f"voxelize Gvox/s at {side}^3", "value": round(nvox / (tf / 1e3) / 1e9, 3), "unit": "Gvox/s",
           "fwd_bwd_gvox_per_s": round(nvox / ((tf + tb) / 1e3) / 1e9, 3), "fwd_ms": round(tf, 4),
           "bwd_ms": round(tb, 4), "steps": k, "voxel_pairs": stats.pixel_pairs,
           "config": {"workload": f"{name}: {n} Gaussians (3D Shepp-Logan phantom cloud) into a {side}^3 grid, "
                                  "voxelize_full (value) and + voxelize_backward with an all-ones grad volume "
                                  "(fwd_bwd_gvox_per_s), device-resident, L2 flushed"},
           "phase_ms_fwd": {p: round(v[0] / k, 4) for p, v in phf.items() if v[1]},
           "phase_ms_bwd": {p: round(v[0] / k, 4) for p, v in phb.items() if v[1]},
           "roofline": roof, "roofline_sfu": sfu}
    if ref is not None:
        cb = cpu_baseline_voxel(ref, cloud_h, side, 64, with_bwd=True)
        out["cpu_baseline"] = {**cb, "value": cb["fwd_gvox_per_s"], "fwd_bwd_gvox_per_s": cb["value"]}
    del vol, gvol, grads, cloud
    torch.cuda.empty_cache()
    return out


def secondary_train(ctx, k: int = 5) -> dict:
    """BASELINE configs[1] as a device-resident training iteration (the loop body of
    train_reconstruction, optim.hpp:456-492, batched over the 75 C2 views): render, fused
    L1 + 0.25 SSIM2D image loss against measured projections (rendered from the unperturbed
    cloud), backward to the Gaussians, the TV term on a 32^3 sub-volume drawn by
    sample_subvolume (voxelize -> tv3d -> voxelize_backward, weight 0.05, added to the
    gradients), lr_schedule for the position rate, one Adam step (batched-gradient data
    parallelism: one optimiser step and one TV sub-volume per 75-view batch)."""
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
    side = WORKLOADS["c2"][0]
    grid = gsct.GridSpec.centered((side, side, side), 1.0)
    rng_sub = gsct.Rng(11)
    extent = gsct.scene_extent(pert)
    horizon = 300 * len(views)  # TrainConfig iterations x views (optim.hpp:435-438)
    vs = gsct.VoxelSettings()

    def it():
        gsct.rasterize_views(st.dcloud, geom, views, st.rs, out=st.images, ctx=ctx)
        lv, _ = gsct.image_loss(st.images, measured, 0.25, grad_out=st.grad_images, ctx=ctx)
        gsct.rasterize_backward_views(st.dcloud, geom, views, st.grad_images, st.rs, out=st.grads, ctx=ctx)
        region = gsct.sample_subvolume(grid, (32, 32, 32), rng_sub)
        sub = gsct.voxelize(st.dcloud, region, vs, ctx=ctx)
        _, tv_grad = gsct.tv3d(sub, ctx=ctx)
        tvg = gsct.voxelize_backward(st.dcloud, region, tv_grad.mul_(0.05), vs, ctx=ctx)
        st.grads.add(tvg)
        lrs.position = gsct.lr_schedule(2e-4 * extent, 1e-6 * extent, adam.step, horizon)
        gsct.adam_step(st.dcloud, adam, st.grads, lrs, ctx=ctx)
        losses.append(float(lv[:, 2].mean()))

    it()
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    ts = timed_steps(it, st.stream, k, lambda: flush.zero_())
    ms = float(np.mean(ts))
    return {"workload": "C2 training iteration: 75 views render + L1/SSIM2D loss + backward + 32^3 TV sub-volume "
                        "(voxelize, tv3d, voxelize_backward) + lr_schedule + Adam (device-resident)",
            "ms_per_iteration": ms, "proj_per_s": len(views) / (ms / 1e3),
            "mean_view_loss_first_last": [losses[0], losses[-1]], "iterations": len(losses)}


def run_dropin(timeout_s: float = 240.0) -> dict:
    """The UNCHANGED reference loop train_reconstruction (optim.hpp:397-538), one epoch at C2
    (75 views at 512^2, 200k Gaussians; per view-step: render, 32^3 TV voxelize, L1+SSIM2D+TV
    loss, backward, voxelize_backward, Adam -- one fwd+bwd projection each), through the C++
    drop-in (oracle/_ref/dropin_train_b200: gsct_b200_dropin.hpp over libgsct_b200.so,
    pageable std::vector buffers; the loop's total_loss_recon on the device too), the same with
    the reference's CPU loss (dropin_train_b200_cpuloss: only the five hot-path operators on
    the GPU), and as the plain reference on the host cores (dropin_train_cpu).
    tests/cpp/dropin_train.cpp."""
    import subprocess

    root = Path(__file__).resolve().parent / "oracle" / "_ref"
    out: dict = {"unit": "view-steps/s (one fwd+bwd projection each) through train_reconstruction",
                 "config": "C2: 200000 Gaussians, 75 cone views at 512^2, 1 epoch, TrainConfig defaults"}
    for tag, exe in (("b200", root / "dropin_train_b200"), ("b200_cpu_loss", root / "dropin_train_b200_cpuloss"),
                     ("cpu", root / "dropin_train_cpu")):
        if not exe.exists():
            out[tag] = {"unavailable": f"{exe.name} not built (needs /root/reference at build time)"}
            continue
        r = subprocess.run([str(exe), "200000", "256", "75", "512", "1"], capture_output=True, text=True,
                           timeout=timeout_s)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        out[tag] = json.loads(line[-1]) if line else {"error": (r.stderr or r.stdout)[-300:]}
    b = out.get("b200", {})
    if "view_steps_per_s" in b:
        out["value"] = b["view_steps_per_s"]
        c = out.get("cpu", {})
        if "view_steps_per_s" in c:
            out["speedup_vs_reference_loop"] = round(b["view_steps_per_s"] / c["view_steps_per_s"], 3)
    return out


def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_2604_01844_b200 import gsct

    torch.cuda.set_device(local_rank)
    ctx = gsct.context(local_rank)
    cloud, geom = make_workload(args.config)
    views = shard_views(len(geom.angles), rank, world)
    # N > 1 over NCCL: the library's own group (one NCCL communicator per context) carries
    # the gradient all-reduce inside gsct_rasterize_bwd; over gloo (ranks sharing one GPU,
    # where NCCL refuses duplicate devices) the packed buffers are reduced by torch
    native = (world > 1 or os.environ.get("GSCT_BENCH_NATIVE_GROUP") == "1") and args.dist_backend == "nccl"
    if native:
        from paper_2604_01844_b200.sharding import native_group

        try:
            native_group(ctx)
        except Exception as exc:  # e.g. NCCL unavailable: the torch reduction carries the sum
            log(f"native group unavailable ({exc}); reducing with torch.distributed")
            native = False
    step = DeviceStep(ctx, cloud, geom, views, world, native_group=native)
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
        e = run_e2e(ctx, cloud, geom, views, max(3, min(args.steps, 5)), 2, world, native_group=native)
        e_ms = float(np.mean(e["ms"]))
        e2e = {"value": round(n_views_total / (e_ms / 1e3), 2), "unit": UNIT, "h2d_bytes_per_step": e["h2d"],
               "d2h_bytes_per_step": e["d2h"], "ms_per_step": round(e_ms, 3),
               "path": "gsct_rasterize_fwd + gsct_rasterize_bwd (C ABI, GSCT_HOST pinned buffers, sync)"
                       + (" with the library's NCCL group (all-reduce inside the backward), max over ranks" if native
                          else " + all-reduce of the packed gradients, max over ranks" if world > 1 else "")}
        ctx.set_async(True)

    if rank != 0:
        return

    peaks = _peaks(ctx)
    n = cloud.size()
    npx = geom.n_u * geom.n_v
    dom = max(("raster_fwd", "raster_bwd"), key=lambda p: phases[p][0])
    bytes_step = len(views) * ((PARAM_B + (GRAD_B if dom == "raster_bwd" else 0)) * n + PX_B * npx)
    roofline, roofline_sfu = roofline_objects(
        peaks, dom, "k_raster_fwd4" if dom == "raster_fwd" else "k_raster_bwd_chain", phases[dom][0],
        phases[dom][1], bytes_step, stats.pixel_pairs, args.steps, "r2/raster" if args.config == "c2" else "-")

    out = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded 3D Shepp-Logan phantom cloud, random init)",
        "config": config_for(args.config, world),
        "work": {"tile_pairs_per_step": stats.tile_pairs, "pixel_pairs_per_pass": stats.pixel_pairs,
                 "culled": stats.culled, "degenerate": stats.degenerate},
        "roofline": roofline, "roofline_sfu": roofline_sfu,
        "phase_ms_per_step": {k: round(v[0] / args.steps, 4) for k, v in phases.items() if v[1]},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    if e2e is not None:
        out["e2e"] = e2e
    if not args.no_secondary and world == 1:
        try:
            out["dropin"] = run_dropin()
        except Exception as exc:
            out["dropin"] = {"error": repr(exc)}
    ref = None
    if not args.no_cpu_baseline and world == 1:
        try:
            from oracle.oracle import Ref

            ref = Ref()
            out["cpu_baseline"] = cpu_baseline_views(ref, cloud, geom, len(geom.angles))
        except Exception as exc:
            out["cpu_baseline"] = {"error": repr(exc)}
    if not args.no_secondary and world == 1:
        sec = {}
        for name, fn in (("raster_2048", lambda: secondary_2k(ctx, peaks, ref)),
                         ("voxel_512", lambda: _voxel_line(ctx, peaks, ref, 512, 500_000, 1, 3, "r2/voxel", "C3")),
                         ("voxel_1024", lambda: _voxel_line(ctx, peaks, ref, 1024, 1_000_000, 1, 2, "r2/voxel_1024",
                                                            "C5 volume")),
                         ("train_iteration_c2", lambda: secondary_train(ctx))):
            try:
                sec[name] = fn()
            except Exception as exc:  # report, never hide the main line
                sec[name] = {"error": repr(exc)}
        out["secondary"] = sec
    print(json.dumps(out), flush=True)


def run_reference(args, rank: int, world: int) -> None:
    """Reference arm: the reference's own CPU implementation (oracle/_ref: the unchanged
    /root/reference headers compiled here) on all host threads, on our arm's workload, metric
    and config. Inputs are built by the reference's Rng / default_geometry (no product
    library is loaded). Each step is a bounded sample of the 75-view step: the first
    calibration view sizes it so the whole --steps/--warmup run stays within a few minutes."""
    if rank != 0:
        return
    from oracle.oracle import REF_LIB, Ref
    from paper_2604_01844_b200.gsct import RasterSettings

    if not REF_LIB.exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libgsct_ref.so was not built"}))
        return
    ref = Ref()
    cores = ref.threads()
    cloud, geom = make_workload_ref(ref, args.config)
    h = ref.cloud(cloud)
    rs = RasterSettings()
    ones = np.ones((geom.n_v, geom.n_u))
    n = cloud.size()
    nv = len(geom.angles)
    cursor = [0]

    def view_pass():
        v = cursor[0] % nv
        cursor[0] += 1
        ref.rasterize_view(h, geom, v, rs)
        ref.rasterize_backward(h, geom, v, ones, rs, n)

    t0 = time.perf_counter()
    view_pass()  # calibration (untimed)
    t_view = time.perf_counter() - t0
    budget_s = float(os.environ.get("GSCT_REF_BUDGET_S", "150"))
    views_per_step = int(max(1, min(nv, budget_s / (max(args.steps + args.warmup, 1) * t_view))))

    def step():
        for _ in range(views_per_step):
            view_pass()

    for _ in range(args.warmup):
        step()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        ts.append((time.perf_counter() - t0) * 1e3)
    ref.free_cloud(h)
    ms = float(np.mean(ts))
    value = views_per_step / (ms / 1e3)
    sample = (f"{views_per_step} of {nv} views fwd+bwd per step (rasterize_view + rasterize_backward, "
              f"projector.hpp:308,371; views cycled), {cores} threads on {cpu_model()}"
              + ("" if views_per_step == nv else "; proj/s per-view rate of the 75-view step"))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded 3D Shepp-Logan phantom cloud, random init)",
        "config": config_for(args.config, world),
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
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
    # GSCT_BENCH_NATIVE_GROUP=1 (under torchrun): the library's NCCL group even at one rank,
    # to exercise the multi-GPU wiring on a one-GPU box
    use_dist = world > 1 or os.environ.get("GSCT_BENCH_NATIVE_GROUP") == "1"
    if use_dist:
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
        if use_dist:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
