"""Per-call wall time of the drop-in's one-view calls (the reference loop's call pattern,
optim.hpp:456-492): pageable host cloud (what the C++ adapter passes) vs pinned vs device."""
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
    variants = {
        "pageable": cloud,
        "pinned": gsct.GaussianCloud(pin(cloud.positions), pin(cloud.log_scales), pin(cloud.rotations),
                                     pin(cloud.raw_densities)),
        "device": cloud.to_device(0),
    }
    grid = gsct.GridSpec.centered((256, 256, 256), 1.0)
    region = gsct.GridRegion.of_parent(grid, (100, 100, 100), (32, 32, 32))
    gimg = np.ones((1, 512, 512), dtype=np.float32)
    gvol = np.ones((32, 32, 32), dtype=np.float32)

    def t(f, reps=10):
        f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            f()
        return (time.perf_counter() - t0) / reps * 1e3

    for name, cl in variants.items():
        row = {
            "fwd": t(lambda: gsct.rasterize_views(cl, geom, [3], ctx=ctx)),
            "bwd": t(lambda: gsct.rasterize_backward_views(cl, geom, [3], gimg, ctx=ctx)),
            "vox32": t(lambda: gsct.voxelize(cl, region, ctx=ctx)),
            "voxbwd32": t(lambda: gsct.voxelize_backward(cl, region, gvol, ctx=ctx)),
        }
        print(name, {k: round(v, 3) for k, v in row.items()}, flush=True)
    a = np.empty(3 * n)
    b = np.empty(3 * n)
    print("host memcpy 4.8MB ms", round(t(lambda: np.copyto(a, b), 20), 3))


if __name__ == "__main__":
    main()
