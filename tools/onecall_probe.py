"""Launch list of single-view calls (the reference loop's call pattern, one view per call) with a
device-resident cloud: which kernels one call launches and how long each runs.
    ncu --metrics gpu__time_duration.sum --csv --log-file out.csv python tools/onecall_probe.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import bench
    from paper_2604_01844_b200 import gsct

    ctx = gsct.context(0)
    cloud, geom = bench.make_workload("c2")
    d = cloud.to_device(0)
    gimg = torch.ones((1, 512, 512), dtype=torch.float32, device="cuda")
    out = torch.empty((1, 512, 512), dtype=torch.float32, device="cuda")
    n = cloud.size()
    grads = gsct.ParamGradients.zeros(n, 0)
    for _ in range(3):
        gsct.rasterize_views(d, geom, [3], out=out, ctx=ctx)
        gsct.rasterize_backward_views(d, geom, [3], gimg, out=grads, ctx=ctx)
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    for _ in range(20):
        gsct.rasterize_views(d, geom, [3], out=out, ctx=ctx)
    t1 = time.perf_counter()
    for _ in range(20):
        gsct.rasterize_backward_views(d, geom, [3], gimg, out=grads, ctx=ctx)
    t2 = time.perf_counter()
    print(f"fwd {1e3 * (t1 - t0) / 20:.3f} ms/call, bwd {1e3 * (t2 - t1) / 20:.3f} ms/call")


if __name__ == "__main__":
    main()
