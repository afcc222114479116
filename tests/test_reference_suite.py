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
