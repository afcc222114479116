"""Builds libgsct_b200.so in-tree (nvcc for sm_100a + g++ for the host harness).

The product's only native artefact. `python -m paper_2604_01844_b200.build_native`
or `__graft_entry__.build()`. Objects go to build/, the library next to this file so
it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libgsct_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
# preprocess.cu holds the fp64 set-up whose operation order must match the reference
# exactly (no FMA contraction) so integer boxes / keys are bit-exact.
PER_FILE = {"preprocess.cu": ["--fmad=false"], "control.cu": ["--fmad=false"], "codec.cu": ["--fmad=false"]}
CU_SOURCES = ["api.cu", "preprocess.cu", "tail.cu", "raster.cu", "order.cu", "voxel.cu", "loss.cu", "control.cu", "codec.cu", "microbench.cu", "group.cu", "hostio.cu"]
CXX_SOURCES = ["host.cpp"]


def _run(cmd: list[str], log: Path) -> None:
    with open(log, "w") as f:
        r = subprocess.run(cmd, stdout=f, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        sys.stderr.write(log.read_text())
        raise RuntimeError(f"build failed: {' '.join(cmd)}")


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_variant(tag: str, defines: list[str]) -> Path:
    """Builds build/variants/libgsct_<tag>.so with extra -D flags (entries starting with '-'
    are passed to nvcc as they are; A/B experiments -- the product library is always the
    default build)."""
    vdir = ROOT / "build" / "variants" / tag
    vdir.mkdir(parents=True, exist_ok=True)
    jobs, objs = [], []
    for src in CU_SOURCES:
        o = vdir / (src + ".o")
        objs.append(o)
        jobs.append(([NVCC] + NVFLAGS + PER_FILE.get(src, []) + [d if d.startswith("-") else f"-D{d}" for d in defines] +
                     ["-c", str(CSRC / src), "-o", str(o)], vdir / (src + ".log")))
    for src in CXX_SOURCES:
        o = vdir / (src + ".o")
        objs.append(o)
        jobs.append((["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-c", str(CSRC / src), "-o", str(o)],
                     vdir / (src + ".log")))
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(lambda j: _run(*j), jobs))
    lib = ROOT / "build" / "variants" / f"libgsct_{tag}.so"
    _run([NVCC] + ARCH + ["-shared", "-o", str(lib)] + [str(o) for o in objs] + ["-ldl"], vdir / "link.log")
    return lib


def build(force: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    headers = sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [ROOT / "include" / "gsct_cuda.h"]
    jobs = []
    objs = []
    for src in CU_SOURCES:
        o = OBJ / (src + ".o")
        objs.append(o)
        if force or _stale(o, [CSRC / src] + headers):
            cmd = [NVCC] + NVFLAGS + PER_FILE.get(src, []) + ["-c", str(CSRC / src), "-o", str(o)]
            jobs.append((cmd, OBJ / (src + ".log")))
    for src in CXX_SOURCES:
        o = OBJ / (src + ".o")
        objs.append(o)
        if force or _stale(o, [CSRC / src] + headers):
            cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-c", str(CSRC / src), "-o", str(o)]
            jobs.append((cmd, OBJ / (src + ".log")))
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        list(ex.map(lambda j: _run(*j), jobs))
    if force or jobs or _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", str(LIB)] + [str(o) for o in objs] + ["-ldl"], OBJ / "link.log")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
