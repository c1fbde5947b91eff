#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep) or launch-list CSV into profiles/*.json.

    python tools/ncu_summary.py report gpurun_out/prof_predict.ncu-rep --rows 100000000 \
        --out profiles/ncu_predict.json --source "..."
    python tools/ncu_summary.py launches gpurun_out/launches.csv --out profiles/launches.json
"""

import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__occupancy_limit_shared_mem": "ctas_per_sm_smem_limit",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active": "fma_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}


def _unit_scale(unit: str) -> float:
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
            "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3,
            "ms": 1e6, "s": 1e9, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}.get(unit, 1.0)


def report(path, rows, out, source):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rd = list(csv.reader(io.StringIO(txt)))
    head, units, vals = rd[0], rd[1], rd[2]
    res = {"kernel": vals[head.index("Kernel Name")], "source": source}
    stalls = {}
    for name, unit, val in zip(head, units, vals):
        try:
            v = float(val.replace(",", ""))
        except ValueError:
            continue
        if name in KEYS:
            res[KEYS[name]] = v * _unit_scale(unit)
        if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith(
                "_per_issue_active.ratio") and v > 0.02:
            stalls[name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
    res["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
    if rows:
        tot = res.get("dram_bytes_read", 0) + res.get("dram_bytes_write", 0)
        res["rows"] = rows
        res["dram_bytes_per_sample"] = tot / rows
        if "duration_ns" in res:
            res["dram_gbs"] = tot / res["duration_ns"]
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


def launches(path, out):
    text = open(path).read()
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rd = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = defaultdict(list)
    for r in rd:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            scale = _unit_scale(r.get("Metric Unit", "nsecond"))
            agg[r["Kernel Name"]].append(float(r["Metric Value"].replace(",", "")) * scale)
    total = sum(sum(v) for v in agg.values())
    res = [{"kernel": k, "launches": len(v), "mean_ns": sum(v) / len(v), "total_ns": sum(v),
            "share": sum(v) / total} for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    for r in res:
        print(f"{r['share']*100:6.2f}%  {r['launches']:3d} x {r['mean_ns']/1e3:10.1f} us  {r['kernel'][:90]}")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=("report", "launches"))
    ap.add_argument("path")
    ap.add_argument("--rows", type=int, default=0)
    ap.add_argument("--out", required=True)
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    report(a.path, a.rows, a.out, a.source) if a.mode == "report" else launches(a.path, a.out)
