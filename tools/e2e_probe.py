"""Where the C-ABI host-buffer (e2e) step spends its time: per call, host vs device buffers."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    import bench
    from paper_2604_01844_b200 import gsct

    ctx = gsct.context(0)
    cloud, geom = bench.make_workload("c2")
    n = cloud.size()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    hc = gsct.GaussianCloud(pin(cloud.positions), pin(cloud.log_scales), pin(cloud.rotations), pin(cloud.raw_densities))
    dc = cloud.to_device(0)
    img_h = torch.empty((75, 512, 512), dtype=torch.float32).pin_memory().numpy()
    gi_h = torch.ones((75, 512, 512), dtype=torch.float32).pin_memory().numpy()
    img_d = torch.empty((75, 512, 512), dtype=torch.float32, device="cuda")
    gi_d = torch.ones((75, 512, 512), dtype=torch.float32, device="cuda")
    z = lambda *s: torch.zeros(s, dtype=torch.float64).pin_memory().numpy()
    gh = gsct.ParamGradients(z(n, 3), z(n, 3), z(n, 4), z(n), z(n), torch.zeros(n, dtype=torch.uint8).pin_memory().numpy())
    gd = gsct.ParamGradients.zeros(n, 0)
    ctx.set_async(False)
    ctx.set_save_for_backward(True)
    rs = gsct.RasterSettings()

    def t(fn, k=5):
        fn()
        ts = []
        for _ in range(k):
            t0 = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t0) * 1e3)
        return round(float(np.median(ts)), 3)

    print("fwd host", t(lambda: gsct.rasterize_views(hc, geom, None, rs, out=img_h, ctx=ctx)))
    print("fwd dev ", t(lambda: gsct.rasterize_views(dc, geom, None, rs, out=img_d, ctx=ctx)))
    gsct.rasterize_views(hc, geom, None, rs, out=img_h, ctx=ctx)
    print("bwd host", t(lambda: (gsct.rasterize_views(hc, geom, None, rs, out=img_h, ctx=ctx),
                                 gsct.rasterize_backward_views(hc, geom, None, gi_h, rs, out=gh, ctx=ctx))))
    print("bwd dev ", t(lambda: (gsct.rasterize_views(dc, geom, None, rs, out=img_d, ctx=ctx),
                                 gsct.rasterize_backward_views(dc, geom, None, gi_d, rs, out=gd, ctx=ctx))))
    x = torch.empty(78643200 // 4, dtype=torch.float32, device="cuda")
    y = torch.empty(78643200 // 4, dtype=torch.float32).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); y.copy_(x); torch.cuda.synchronize(); print("D2H 78.6MB ms", (time.perf_counter() - t0) * 1e3)
    t0 = time.perf_counter(); x.copy_(y); torch.cuda.synchronize(); print("H2D 78.6MB ms", (time.perf_counter() - t0) * 1e3)


if __name__ == "__main__":
    main()
