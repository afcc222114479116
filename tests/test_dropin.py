"""GPU: the C++ drop-in parity suite (tests/cpp/dropin_parity.cpp, prebuilt into
oracle/_ref/dropin_parity): the reference's own types, fixtures, training loops
(train_reconstruction, train_volume_fit) and bench sweep running unchanged on the B200
operators through the C++ adapter, checked against the reference CPU operators in-process."""
from __future__ import annotations

import subprocess

import pytest

from conftest import ROOT

EXE = ROOT / "oracle" / "_ref" / "dropin_parity"


@pytest.mark.gpu
def test_dropin_parity_suite(ctx):
    if not EXE.exists():
        pytest.skip("oracle/_ref/dropin_parity not built (needs /root/reference at build time)")
    out = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, (out.stdout[-2000:], out.stderr[-4000:])
    assert "| 0 failed" in out.stdout
