"""C5 voxelization: 1M-Gaussian Shepp-Logan cloud into a 1024^3 grid, fwd + bwd timing."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    from paper_2604_01844_b200 import gsct

    side, n = 1024, 1_000_000
    ctx = gsct.context(0)
    cloud = gsct.make_cloud("shepp_logan", n, seed=2, side=side, spacing=1.0).to_device(0)
    grid = gsct.GridSpec.centered((side,) * 3, 1.0)
    region = gsct.GridRegion.covering(grid)
    vol = torch.empty((side,) * 3, dtype=torch.float32, device="cuda")
    gvol = torch.ones_like(vol)
    grads = gsct.ParamGradients.zeros(n, 0)
    st = gsct.RenderStats()
    gsct.voxelize(cloud, region, gsct.VoxelSettings(), st, out=vol, ctx=ctx)
    ctx.set_async(True)
    ctx.set_profiling(True)
    ctx.phase_times()
    for _ in range(3):
        gsct.voxelize(cloud, region, out=vol, ctx=ctx)
        gsct.voxelize_backward(cloud, region, gvol, out=grads, ctx=ctx)
    ph = {k: round(v[0] / 3, 3) for k, v in ctx.phase_times().items() if v[1]}
    fwd = ph["voxel_setup"] / 2 + ph["voxel_bin"] + ph["voxel_fwd"]
    print(ph, "pairs", st.pixel_pairs, "fwd Gvox/s ~", side ** 3 / (fwd / 1e3) / 1e9)


if __name__ == "__main__":
    main()
