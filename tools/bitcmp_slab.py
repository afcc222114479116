"""z-slab vs full volume, bitwise, for every built variant (debug helper)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

if len(sys.argv) > 1 and sys.argv[1] == "dump":
    from paper_2604_01844_b200 import gsct
    cloud = gsct.make_cloud("random", 80, seed=60, pos_range=6.0)
    grid = gsct.GridSpec.centered((30, 28, 37), 0.5)
    region = gsct.GridRegion.covering(grid)
    full = gsct.voxelize(cloud, region)
    cuts = [0, 9, 10, 24, 37]
    slabs = np.concatenate([gsct.voxelize(cloud, region, window=((0, 0, a), (30, 28, b)))
                            for a, b in zip(cuts, cuts[1:])], axis=0)
    np.savez(sys.argv[2], full=full, slabs=slabs)
else:
    libs = sorted((ROOT / "build" / "variants").glob("libgsct_*.so"))
    outs = {}
    for lib in libs:
        o = f"/tmp/{lib.stem}_slab.npz"
        subprocess.run([sys.executable, __file__, "dump", o], env=dict(os.environ, GSCT_LIB_PATH=str(lib)), check=True)
        outs[lib.stem] = np.load(o)
    for k, v in outs.items():
        d = v["full"] != v["slabs"]
        print(k, "slab==full", np.array_equal(v["full"], v["slabs"]), "n diff", int(d.sum()),
              "where z", sorted(set(np.nonzero(d)[0].tolist()))[:10])
    ks = list(outs)
    print("full old==new", np.array_equal(outs[ks[0]]["full"], outs[ks[1]]["full"]),
          "slabs old==new", np.array_equal(outs[ks[0]]["slabs"], outs[ks[1]]["slabs"]))
