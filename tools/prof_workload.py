"""Runs one device-resident pass of a benchmark workload for ncu captures.

    python tools/prof_workload.py raster c2     # rasterize fwd + bwd of the C2 workload
    python tools/prof_workload.py voxel c3      # voxelize_full + voxelize_backward at 512^3

Each phase runs twice (the first is a warm-up), so `ncu -k regex:<kernel> -s 1 -c 1`
captures a warm launch. Prints per-phase device ms measured with CUDA events.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    import torch

    import bench
    from paper_2604_01844_b200 import gsct

    what = sys.argv[1] if len(sys.argv) > 1 else "raster"
    cfg = sys.argv[2] if len(sys.argv) > 2 else ("c2" if what == "raster" else "c3")
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    ctx = gsct.context(0)
    ctx.set_async(True)
    ctx.set_profiling(True)
    if what == "e2e":  # C-ABI host-buffer fwd / fwd+bwd wall times (sync calls), ms
        import time

        import numpy as np
        cloud, geom = bench.make_workload(cfg)
        n, nv = cloud.size(), len(geom.angles)
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        hc = gsct.GaussianCloud(pin(cloud.positions), pin(cloud.log_scales), pin(cloud.rotations),
                                pin(cloud.raw_densities))
        img = torch.empty((nv, geom.n_v, geom.n_u), dtype=torch.float32).pin_memory().numpy()
        gi = torch.ones((nv, geom.n_v, geom.n_u), dtype=torch.float32).pin_memory().numpy()
        z = lambda *s: torch.zeros(s, dtype=torch.float64).pin_memory().numpy()
        gh = gsct.ParamGradients(z(n, 3), z(n, 3), z(n, 4), z(n), z(n),
                                 torch.zeros(n, dtype=torch.uint8).pin_memory().numpy())
        ctx.set_async(False)
        ctx.set_profiling(False)
        ctx.set_save_for_backward(True)
        rs = gsct.RasterSettings()

        def med(fn, k=int(reps) * 3):
            fn()
            ts = []
            for _ in range(k):
                t0 = time.perf_counter()
                fn()
                ts.append((time.perf_counter() - t0) * 1e3)
            return round(float(np.median(ts)), 3)

        fwd = med(lambda: gsct.rasterize_views(hc, geom, None, rs, out=img, ctx=ctx))
        both = med(lambda: (gsct.rasterize_views(hc, geom, None, rs, out=img, ctx=ctx),
                            gsct.rasterize_backward_views(hc, geom, None, gi, rs, out=gh, ctx=ctx)))
        print(json.dumps({"fwd_host_ms": fwd, "fwdbwd_host_ms": both, "proj_per_s": round(nv / both * 1e3, 1)}))
        return
    if what == "raster":
        cloud, geom = bench.make_workload(cfg)
        step = bench.DeviceStep(ctx, cloud, geom, list(range(len(geom.angles))), 1)
        step()  # warm-up (workspace allocation), excluded from the phase times
        ctx.phase_times()
        for _ in range(reps):
            step()
    else:
        side, n = {"c3": (512, 500_000), "c5": (1024, 1_000_000)}.get(cfg, (128, 50_000))
        cloud = gsct.make_cloud("shepp_logan", n, seed=1, side=side, spacing=1.0).to_device(0)
        region = gsct.GridRegion.covering(gsct.GridSpec.centered((side, side, side), 1.0))
        vol = torch.empty((side, side, side), dtype=torch.float32, device="cuda")
        gvol = torch.ones_like(vol)
        grads = gsct.ParamGradients.zeros(n, 0)
        gsct.voxelize(cloud, region, out=vol, ctx=ctx)
        gsct.voxelize_backward(cloud, region, gvol, out=grads, ctx=ctx)
        ctx.phase_times()
        for _ in range(reps):
            gsct.voxelize(cloud, region, out=vol, ctx=ctx)
            gsct.voxelize_backward(cloud, region, gvol, out=grads, ctx=ctx)
    ph = ctx.phase_times()
    print(json.dumps({k: round(v[0] / reps, 4) for k, v in ph.items() if v[1]}))


if __name__ == "__main__":
    main()
