"""Summarises ncu captures (gpurun_out/*.ncu-rep, launch-list CSVs) into profiles/<tag>/.

    python tools/ncu_summary.py <tag> <glob-of-ncu-rep> [launches.csv]

Writes profiles/<tag>/summary.json (per kernel: duration, DRAM bytes, pipe utilisation,
issue activity, occupancy, top stall reasons), profiles/<tag>/summary.md and, when given,
profiles/<tag>/launches.csv (the --metrics gpu__time_duration.sum launch list).
"""
from __future__ import annotations

import csv
import glob
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1.0),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "xu_pipe_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1.0),
    "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "alu_pipe_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "inst_executed": ("smsp__inst_executed.sum", 1.0),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1.0),
    "sm_clock_hz": ("sm__cycles_elapsed.avg.per_second", None),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "l1tex_throughput_pct": ("l1tex__throughput.avg.pct_of_peak_sustained_active", 1.0),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "l1_lsu_wavefronts_pct": ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 1.0),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ms": 1.0, "us": 1e-3, "ns": 1e-6,
              "s": 1e3, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def raw(rep: str) -> tuple[list[str], list[str], list[list[str]]]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def kname(full: str) -> str:
    """Bare kernel name: text before the first template/argument list, last scope."""
    full = full.replace("<unnamed>", "anon").replace("(anonymous namespace)", "anon")
    cut = min([i for i in (full.find("<"), full.find("(")) if i >= 0] or [len(full)])
    return full[:cut].replace("void ", "").split("::")[-1].strip()


def summarise_row(h: list[str], units: list[str], v: list[str], stem: str) -> dict:
    d = {"kernel": kname(v[h.index("Kernel Name")]) if "Kernel Name" in h else stem}
    for key, (metric, _) in METRICS.items():
        if metric in h:
            i = h.index(metric)
            try:
                x = float(v[i].replace(",", ""))
            except ValueError:
                continue
            d[key] = x * UNIT_SCALE.get(units[i], 1.0)
    stalls = {}
    for i, name in enumerate(h):
        if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
            try:
                stalls[name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v[i])
            except ValueError:
                pass
    d["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:5])
    if "dram_read_bytes" in d and "dram_write_bytes" in d:
        d["dram_bytes"] = d["dram_read_bytes"] + d["dram_write_bytes"]
    return d


def summarise(rep: str) -> list[dict]:
    """One entry per captured launch of the report."""
    h, units, vals = raw(rep)
    return [summarise_row(h, units, v, Path(rep).stem) for v in vals if len(v) == len(h)]


def launch_shares(path: str) -> list[tuple[str, int, float]]:
    """(kernel, launches, total ms) from a --metrics gpu__time_duration.sum launch list."""
    agg: dict[str, list] = {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = kname(r["Kernel Name"])
        ms = float(r["Metric Value"].replace(",", "")) * UNIT_SCALE.get(r["Metric Unit"], 1e-6)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    return sorted(((k, v[0], v[1]) for k, v in agg.items()), key=lambda t: -t[2])


def main() -> None:
    tag = sys.argv[1]
    reps = sorted(glob.glob(sys.argv[2]))
    out = ROOT / "profiles" / tag
    out.mkdir(parents=True, exist_ok=True)
    rows = [d for r in reps for d in summarise(r)]
    (out / "summary.json").write_text(json.dumps(rows, indent=1))
    lines = ["| kernel | ms (ncu) | DRAM MB | issue % | L1 % | L2 % | XU % | FMA % | ALU % | FP64 % | warps % | regs | top stall |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for d in rows:
        top = next(iter(d["top_stalls"].items()), ("-", 0))
        lines.append(f"| {d['kernel']} | {d.get('duration_ms', 0):.3f} | {d.get('dram_bytes', 0) / 1e6:.1f} | "
                     f"{d.get('issue_active_pct', 0):.1f} | {d.get('l1tex_throughput_pct', 0):.1f} | "
                     f"{d.get('l2_throughput_pct', 0):.1f} | {d.get('xu_pipe_pct', 0):.1f} | {d.get('fma_pipe_pct', 0):.1f} | "
                     f"{d.get('alu_pipe_pct', 0):.1f} | {d.get('fp64_pipe_pct', 0):.1f} | {d.get('warps_active_pct', 0):.1f} | "
                     f"{int(d.get('registers', 0))} | {top[0]} {top[1]:.2f} |")
    if len(sys.argv) > 3:
        shutil.copy(sys.argv[3], out / "launches.csv")
        sh = launch_shares(sys.argv[3])
        tot = sum(t[2] for t in sh) or 1.0
        lines += ["", "Launch list (`--metrics gpu__time_duration.sum --clock-control none`, cold-cache, serialised):", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        lines += [f"| {k} | {c} | {ms:.3f} | {100 * ms / tot:.1f}% |" for k, c, ms in sh]
    (out / "summary.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
