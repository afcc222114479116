import sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
from paper_2604_01844_b200 import gsct
ctx = gsct.context(0)
cloud, geom = bench.make_workload("c2")
n, nv = cloud.size(), len(geom.angles)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
hc = gsct.GaussianCloud(pin(cloud.positions), pin(cloud.log_scales), pin(cloud.rotations), pin(cloud.raw_densities))
img = torch.empty((nv, geom.n_v, geom.n_u), dtype=torch.float32).pin_memory().numpy()
gi = torch.ones((nv, geom.n_v, geom.n_u), dtype=torch.float32).pin_memory().numpy()
z = lambda *s: torch.zeros(s, dtype=torch.float64).pin_memory().numpy()
gh = gsct.ParamGradients(z(n, 3), z(n, 3), z(n, 4), z(n), z(n), torch.zeros(n, dtype=torch.uint8).pin_memory().numpy())
ctx.set_save_for_backward(True)
rs = gsct.RasterSettings()
for prof in (False, True):
    ctx.set_profiling(prof)
    for _ in range(3):
        gsct.rasterize_views(hc, geom, None, rs, out=img, ctx=ctx); gsct.rasterize_backward_views(hc, geom, None, gi, rs, out=gh, ctx=ctx)
    ctx.phase_times()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        t1 = time.perf_counter(); gsct.rasterize_views(hc, geom, None, rs, out=img, ctx=ctx); t2 = time.perf_counter()
        gsct.rasterize_backward_views(hc, geom, None, gi, rs, out=gh, ctx=ctx); t3 = time.perf_counter()
        ts.append(((t2 - t1) * 1e3, (t3 - t2) * 1e3))
    ph = ctx.phase_times()
    print("profiling", prof, "fwd/bwd wall ms", np.median([a for a, b in ts]), np.median([b for a, b in ts]))
    if prof: print(json.dumps({k: round(v[0] / 10, 4) for k, v in ph.items() if v[1]}))
