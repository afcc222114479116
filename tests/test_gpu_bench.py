"""The bench.py contract (the driver parses its last stdout line): one JSON object with the
headline metric on the C2 workload, the roofline / cpu_baseline / e2e / clocks /
gpu_launches keys, and internally consistent numbers. Runs the real bench on the GPU with
the secondary lines and the CPU baseline switched off (they are exercised by the driver's
own bench run)."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def test_bench_line_contract():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3", "--no-secondary",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3 and line["higher_is_better"] is True
    assert line["unit"] == "projections/s" and line["value"] > 0 and line["ms_per_step"] > 0
    # value = 75 projections per step / step time
    assert abs(line["value"] - 75 / (line["ms_per_step"] / 1e3)) / line["value"] < 0.02
    assert "workload" in line["config"] and "C2" in line["config"]["workload"]
    roof = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in roof, k
    assert roof["bound"] in ("hbm", "tensor") and 0 < roof["frac"] < 1
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-3
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["unit"] == line["unit"]
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert e2e["value"] <= line["value"] * 1.05  # host copies inside the timed region cost time
    assert line["gpu_launches"] > 0
    assert line["clocks"]["sm_mhz"] > 0
