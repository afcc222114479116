"""A/B timing of compile-time kernel variants.

Here (CPU):   python tools/ab_variants.py build name1=DEF1,DEF2 name2=...
GPU box:      python tools/ab_variants.py run raster c2        (times every built variant)

Each variant is a full libgsct build under build/variants/ loaded through GSCT_LIB_PATH in
a fresh process running tools/prof_workload.py, so per-phase device times are comparable.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    cmd = sys.argv[1]
    if cmd == "build":
        from paper_2604_01844_b200 import build_native

        for spec in sys.argv[2:]:
            tag, _, defs = spec.partition("=")
            lib = build_native.build_variant(tag, [d for d in defs.split(",") if d])
            print(tag, lib)
    elif cmd == "run":
        what = sys.argv[2] if len(sys.argv) > 2 else "raster"
        cfg = sys.argv[3] if len(sys.argv) > 3 else "c2"
        reps = sys.argv[4] if len(sys.argv) > 4 else "3"
        libs = sorted((ROOT / "build" / "variants").glob("libgsct_*.so"))
        for lib in libs:
            env = dict(os.environ, GSCT_LIB_PATH=str(lib))
            out = subprocess.run([sys.executable, str(ROOT / "tools" / "prof_workload.py"), what, cfg, reps],
                                 env=env, capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            print(f"{lib.stem:28s} {line}", flush=True)


if __name__ == "__main__":
    main()
