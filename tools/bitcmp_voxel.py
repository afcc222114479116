"""Bitwise comparison of voxelize outputs between two builds (GSCT_LIB_PATH per process)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

if len(sys.argv) > 1 and sys.argv[1] == "dump":
    import torch

    from paper_2604_01844_b200 import gsct
    out = sys.argv[2]
    res = {}
    for side, n in ((128, 50_000), (512, 500_000)):
        cloud = gsct.make_cloud("shepp_logan", n, seed=1, side=side, spacing=1.0).to_device(0)
        region = gsct.GridRegion.covering(gsct.GridSpec.centered((side, side, side), 1.0))
        vol = torch.empty((side, side, side), dtype=torch.float32, device="cuda")
        gsct.voxelize(cloud, region, out=vol)
        res[f"v{side}"] = vol.cpu().numpy()
    np.savez(out, **res)
else:
    libs = sorted((ROOT / "build" / "variants").glob("libgsct_*.so"))
    outs = []
    for lib in libs:
        o = f"/tmp/{lib.stem}.npz"
        subprocess.run([sys.executable, __file__, "dump", o], env=dict(os.environ, GSCT_LIB_PATH=str(lib)), check=True)
        outs.append(np.load(o))
    for k in outs[0].files:
        print(k, [np.array_equal(outs[0][k], o[k]) for o in outs[1:]], [lib.stem for lib in libs])
