"""Summarise ncu captures into profiles/ (tracked).

    python tools/ncu_summary.py --round r01 \
        --rep k_validate=gpurun_out/prof_k_validate.ncu-rep \
        --rep k_batch=gpurun_out/prof_k_batch.ncu-rep \
        --launches gpurun_out/launches.csv

Writes profiles/ncu_summary.json (read by bench.py for roofline.traffic) and
profiles/<round>_ncu_<kernel>.json / <round>_launches.json.  `ncu -i` runs
here (no GPU needed to read a report).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "alu_pipe_pct_active": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fmaheavy_pipe_pct_active": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "inst_executed": "sm__inst_executed.sum",
    "registers_per_thread": "launch__registers_per_thread",
    "grid_size": "launch__grid_size",
    "block_size": "launch__block_size",
    "sm_clock_hz": "smsp__cycles_elapsed.avg.per_second",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3,
              "s": 1e6, "Mhz": 1e6, "Ghz": 1e9, "hz": 1, "Khz": 1e3}


def raw(rep: Path) -> tuple[list[str], list[str], list[str]]:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def num(v: str, unit: str) -> float | None:
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * UNIT_SCALE.get(unit, 1)


def summarise(rep: Path) -> dict:
    h, u, v = raw(rep)
    col = {name: i for i, name in enumerate(h)}
    s: dict = {"report": rep.name, "kernel_name": v[col["Kernel Name"]] if "Kernel Name" in col else None}
    for key, m in METRICS.items():
        if m in col:
            s[key] = num(v[col[m]], u[col[m]])
    if s.get("dram_read_bytes") is not None and s.get("dram_write_bytes") is not None:
        s["dram_bytes_per_launch"] = s["dram_read_bytes"] + s["dram_write_bytes"]
    stalls = {}
    for name, i in col.items():
        if name.startswith("smsp__average_warp_latency_issue_stalled_") and name.endswith(".ratio"):
            x = num(v[i], u[i])
            if x:
                stalls[name[len("smsp__average_warp_latency_issue_stalled_"):-len(".ratio")]] = x
    if not stalls:
        for name, i in col.items():
            if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("_not_issued"):
                x = num(v[i], u[i])
                if x:
                    stalls[name[len("smsp__pcsamp_warps_issue_stalled_"):]] = x
    s["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
    return s


def launches(path: Path) -> dict:
    rows = list(csv.reader(path.open()))
    hdr = None
    per = defaultdict(lambda: {"count": 0, "total_us": 0.0})
    for r in rows:
        if hdr is None:
            if "Kernel Name" in r and "Metric Value" in r:
                hdr = {k: i for i, k in enumerate(r)}
            continue
        if len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[hdr["Kernel Name"]].split("(")[0]
        val = num(r[hdr["Metric Value"]], r[hdr["Metric Unit"]]) or 0.0
        per[name]["count"] += 1
        per[name]["total_us"] += val
    tot = sum(p["total_us"] for p in per.values()) or 1.0
    out = {k: {**p, "mean_us": p["total_us"] / p["count"], "share": p["total_us"] / tot}
           for k, p in sorted(per.items(), key=lambda kv: -kv[1]["total_us"])}
    return {"source": path.name, "metric": "gpu__time_duration.sum (--clock-control none, serialised, cold)",
            "kernels": out}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--rep", action="append", default=[], help="kernel=path.ncu-rep")
    ap.add_argument("--launches")
    ap.add_argument("--command", default="python bench.py")
    a = ap.parse_args()
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    summary_path = prof / "ncu_summary.json"
    summary = json.loads(summary_path.read_text()) if summary_path.exists() else {"kernels": {}}
    for spec in a.rep:
        kernel, path = spec.split("=", 1)
        s = summarise(Path(path))
        s["command"] = a.command
        s["round"] = a.round
        (prof / f"{a.round}_ncu_{kernel}.json").write_text(json.dumps(s, indent=1) + "\n")
        summary["kernels"][kernel] = s
        print(kernel, json.dumps({k: s.get(k) for k in ("duration_us", "dram_bytes_per_launch",
                                                         "alu_pipe_pct_active", "issue_active_pct")}))
    if a.launches:
        l = launches(Path(a.launches))
        l["command"] = a.command
        (prof / f"{a.round}_launches.json").write_text(json.dumps(l, indent=1) + "\n")
        summary["launches"] = f"{a.round}_launches.json"
        for k, p in l["kernels"].items():
            print(f"  {k}: n={p['count']} mean={p['mean_us']:.1f}us share={p['share']:.3f}")
    summary["source"] = f"{a.round} ncu --set full capture, scripts/gpu_profile.sh"
    summary_path.write_text(json.dumps(summary, indent=1) + "\n")


if __name__ == "__main__":
    main()
