"""Bitwise comparison of C2 forward images and backward gradients between built variants."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

if len(sys.argv) > 1 and sys.argv[1] == "dump":
    import torch

    import bench
    from paper_2604_01844_b200 import gsct
    cloud, geom = bench.make_workload("c2")
    d = cloud.to_device(0)
    img = gsct.rasterize_views(d, geom)
    gi = torch.sin(img * 3.0)
    g = gsct.rasterize_backward_views(d, geom, None, gi)
    np.savez(sys.argv[2], img=img.cpu().numpy(), gpos=g.positions.cpu().numpy(), gls=g.log_scales.cpu().numpy())
else:
    libs = sorted((ROOT / "build" / "variants").glob("libgsct_*.so"))
    outs = []
    for lib in libs:
        o = f"/tmp/{lib.stem}_r.npz"
        subprocess.run([sys.executable, __file__, "dump", o], env=dict(os.environ, GSCT_LIB_PATH=str(lib)), check=True)
        outs.append(np.load(o))
    for k in outs[0].files:
        print(k, [np.array_equal(outs[0][k], o[k]) for o in outs[1:]], [lib.stem for lib in libs])
