"""Shared fixtures. `-m gpu` tests need a B200 (they call the CUDA path through the C ABI);
everything else runs on CPU (oracle vs reference, golden vectors, host logic, gloo)."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_2604_01844_b200 import gsct  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libgsct_b200.so")
    config.addinivalue_line("markers", "slow: larger parity sizes")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Orc

    return Orc()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_LIB, Ref

    if not REF_LIB.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Ref()


@pytest.fixture(scope="session")
def ctx():
    if not has_gpu():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return gsct.context(0)


def parallel_geometry(n: int, spacing: float, angles) -> gsct.ScanGeometry:
    """test_projector.cpp:10-17"""
    return gsct.ScanGeometry("parallel", n, n, spacing, spacing, list(angles))


def cone_geometry(n: int, spacing: float, angles, so: float = 50.0, od: float = 25.0) -> gsct.ScanGeometry:
    return gsct.ScanGeometry("cone", n, n, spacing, spacing, list(angles), so, od)


def oracle_settings() -> gsct.RasterSettings:
    """test_projector.cpp:20-27: no dilation, wide 6-sigma bounds."""
    return gsct.RasterSettings(tau_cut=1e-12, sigma_cap=6.0, dilate=False)


def max_err_rel_peak(a, b) -> float:
    """oracles.hpp:141-149"""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    peak = np.max(np.abs(b)) if b.size else 0.0
    if peak == 0.0:
        peak = 1.0
    return float(np.max(np.abs(a - b)) / peak) if a.size else 0.0


def grad_class_errors(gpu: gsct.ParamGradients, ref: dict) -> dict:
    """Per parameter class: max|d| / max|g_ref| (SURVEY.md App. A.3 gate)."""
    out = {}
    for name in ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm"):
        g = np.asarray(getattr(gpu, name) if not isinstance(gpu, dict) else gpu[name], dtype=np.float64)
        r = np.asarray(ref[name], dtype=np.float64)
        scale = np.max(np.abs(r)) if r.size else 0.0
        out[name] = float(np.max(np.abs(g - r)) / scale) if scale > 0 else float(np.max(np.abs(g - r), initial=0.0))
    return out


def ones_like_image(geom, views=1):
    return np.ones((views, geom.n_v, geom.n_u), dtype=np.float32)
