"""Device time of one fwd+bwd step vs the sum of its profiled phases (finds un-phased gaps).

    python tools/step_gaps.py c5 [views]
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    from paper_2604_01844_b200 import gsct

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
    cloud, geom = bench.make_workload(cfg)
    nv = int(sys.argv[2]) if len(sys.argv) > 2 else len(geom.angles)
    ctx = gsct.context(0)
    ctx.set_async(True)
    st = bench.DeviceStep(ctx, cloud, geom, list(range(nv)), 1)
    st()
    st()
    torch.cuda.synchronize()
    for prof in (False, True):
        ctx.set_profiling(prof)
        ctx.phase_times()
        ts = bench.timed_steps(st, st.stream, 3, lambda: None)
        ph = ctx.phase_times()
        tot = sum(v[0] for v in ph.values()) / 3
        print(json.dumps({"cfg": cfg, "views": nv, "profiling": prof, "step_ms": [round(t, 2) for t in ts],
                          "phase_sum_ms": round(tot, 2),
                          "phases": {k: round(v[0] / 3, 2) for k, v in ph.items() if v[1]}}), flush=True)


if __name__ == "__main__":
    main()
