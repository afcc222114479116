"""The reference's OWN hot-path test executables (test_core, test_projector,
test_voxelizer, test_bench, and test_losses for the next-row image loss, from
/root/reference/proj/tests), compiled unchanged with the test-only Eigen/Catch2 shims into
oracle/_ref/. All 50 test cases must pass: this pins the
shims (and therefore the restatement oracle, which equals the reference bit for bit, see
test_oracle_vs_ref.py) against the reference's known answers and fixtures."""
from __future__ import annotations

import subprocess

import pytest

from conftest import ROOT

REF = ROOT / "oracle" / "_ref"


@pytest.mark.parametrize("name,cases", [("test_core", 10), ("test_projector", 17), ("test_voxelizer", 11),
                                        ("test_bench", 5), ("test_losses", 7)])
def test_reference_suite_passes(name, cases):
    exe = REF / name
    if not exe.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert f"test cases: {cases} | {cases} passed | 0 failed" in out.stdout


def test_reference_optim_suite():
    """test_optim (Adam, lr schedule, adaptive control, training loops) of the unchanged
    reference: 15 of 16 cases pass. The one failure is the reference's own: "adaptive_control
    clones small high-gradient splats with a nudge" (test_optim.cpp:189-207) draws splat 0 of
    random_cloud(75, 3) with scales (0.748, 2.221, 2.056); 2.221 >= split_scale_fraction 0.01 x
    scene_extent 100 = 1.0, so adaptive_control (optim.hpp:232-239) SPLITS it while the test
    expects a clone. The device adaptive control reproduces the split (test_next_ops.py)."""
    exe = REF / "test_optim"
    if not exe.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert "test cases: 16 | 15 passed | 1 failed" in out.stdout
    failed = [ln for ln in (out.stdout + out.stderr).splitlines() if "FAILED" in ln]
    assert failed and all("clones small high-gradient splats with a nudge" in ln for ln in failed), failed
