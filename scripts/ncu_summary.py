#!/usr/bin/env python
"""Summarise the ncu captures brought back in gpurun_out/ into profiles/.

  python scripts/ncu_summary.py <round-tag>      e.g. r01

For every gpurun_out/prof_<w>.ncu-rep (one `ncu --set full` capture of the
top kernel) writes profiles/<tag>/ncu_<w>.txt (the metrics the roofline and
DESIGN.md cite) and profiles/traffic_<w>.json (dram read+write bytes per
launch, read by bench.py for roofline.traffic).  For every
gpurun_out/launches_<w>.csv (the `--metrics gpu__time_duration.sum` launch
list) writes profiles/<tag>/launches_<w>.txt: per-kernel count, mean and
share of device time.
"""
from __future__ import annotations

import collections
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__cluster_dim_x", "launch__shared_mem_per_block_dynamic",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def unit_bytes(v: str, u: str) -> float:
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def summarise_rep(path, tag):
    w = os.path.basename(path)[len("prof_"):-len(".ncu-rep")]
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return
    h, units = rows[0], rows[1]
    lines, traffic = [], []
    for r in rows[2:]:
        for k in KEYS:
            if k in h:
                i = h.index(k)
                lines.append(f"{k:70s} {r[i]} {units[i]}")
        rd = unit_bytes(r[h.index("dram__bytes_read.sum")], units[h.index("dram__bytes_read.sum")])
        wr = unit_bytes(r[h.index("dram__bytes_write.sum")], units[h.index("dram__bytes_write.sum")])
        traffic.append(rd + wr)
        lines.append("")
    d = os.path.join(ROOT, "profiles", tag)
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, f"ncu_{w}.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none capture ({os.path.basename(path)})\n")
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(ROOT, "profiles", f"traffic_{w}.json"), "w") as f:
        json.dump({"dram_bytes_per_launch": int(sum(traffic) / len(traffic)), "source":
                   f"profiles/{tag}/ncu_{w}.txt (dram__bytes_read.sum + dram__bytes_write.sum)"}, f)


def summarise_launches(path, tag):
    w = os.path.basename(path)[len("launches_"):-len(".csv")]
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        return
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    d = collections.defaultdict(list)
    unit = "ns"
    for r in rows[1:]:
        try:
            d[r[ki]].append(float(r[vi].replace(",", "")))
            unit = r[ui]
        except ValueError:
            pass
    tot = sum(sum(v) for v in d.values())
    out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list ({w});",
           "# cold-cache, serialised: compare shares, not absolutes", ""]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"n={len(v):4d} mean={sum(v) / len(v):10.1f} {unit} share={sum(v) / tot:6.3f}  {k}")
    dd = os.path.join(ROOT, "profiles", tag)
    os.makedirs(dd, exist_ok=True)
    with open(os.path.join(dd, f"launches_{w}.txt"), "w") as f:
        f.write("\n".join(out) + "\n")


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    for p in sorted(glob.glob(os.path.join(OUT, "prof_*.ncu-rep"))):
        summarise_rep(p, tag)
    for p in sorted(glob.glob(os.path.join(OUT, "launches_*.csv"))):
        summarise_launches(p, tag)


if __name__ == "__main__":
    main()
