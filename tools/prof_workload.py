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
    if what == "raster":
        cloud, geom = bench.make_workload(cfg)
        step = bench.DeviceStep(ctx, cloud, geom, list(range(len(geom.angles))), 1)
        step()  # warm-up (workspace allocation), excluded from the phase times
        ctx.phase_times()
        for _ in range(reps):
            step()
    else:
        side, n = (512, 500_000) if cfg == "c3" else (128, 50_000)
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
