"""Summarise ncu captures into profiles/ (run here, on the CPU box, after a gpurun).

  python tools/ncu_summary.py gpurun_out/prof_svd_small.ncu-rep <tag>   # --set full capture
  python tools/ncu_summary.py --launches gpurun_out/launches_chi16.csv <tag>

Writes profiles/<tag>.md (key metrics) and merges per-launch DRAM traffic into
profiles/ncu_traffic.json (bench.py reads it for roofline.traffic).
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = "/usr/local/cuda/bin/ncu"
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active", "smsp__average_warp_latency_issue_stalled_barrier",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
    "launch__grid_size", "launch__block_size", "sm__maximum_warps_per_active_cycle_pct",
]


def raw(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def stalls(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "details", "--csv", "--section", "WarpStateStats"],
                         capture_output=True, text=True).stdout
    return out


def summarise_full(rep, tag):
    hdr, units, data = raw(rep)
    lines = ["# ncu summary: %s" % tag, "", "capture: `%s` (ncu --set full --clock-control none)" % os.path.basename(rep), ""]
    traffic = {}
    for row in data:
        rec = dict(zip(hdr, row))
        name = rec.get("Kernel Name", "?")
        lines.append("## %s" % name)
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k in KEYS:
            if k in rec:
                lines.append("| %s | %s | %s |" % (k, rec[k], units[hdr.index(k)]))
        lines.append("")
        try:
            rb = float(rec["dram__bytes_read.sum"].replace(",", ""))
            wb = float(rec["dram__bytes_write.sum"].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rb *= scale.get(units[hdr.index("dram__bytes_read.sum")], 1)
            wb *= scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
            traffic[name] = rb + wb
        except (KeyError, ValueError):
            pass
    st = stalls(rep)
    if st:
        lines += ["## warp state (stall reasons)", "", "```", st.strip()[:6000], "```", ""]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", tag + ".md"), "w").write("\n".join(lines) + "\n")
    return traffic


def summarise_launches(path, tag):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    per = {}
    for r in rows[hdr_i + 1:]:
        if len(r) != len(hdr):
            continue
        rec = dict(zip(hdr, r))
        if rec.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = rec["Kernel Name"].split("(")[0]
        try:
            v = float(rec["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        unit = rec.get("Metric Unit", "nsecond")
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(unit, 1e-3)
        c, t = per.get(name, (0, 0.0))
        per[name] = (c + 1, t + v)
    tot = sum(t for _, t in per.values())
    lines = ["# launch list: %s" % tag, "", "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised:"
             " compare SHARES, not absolutes)", "", "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append("| %s | %d | %.1f | %.1f%% |" % (name, c, t, 100 * t / tot if tot else 0))
    open(os.path.join(ROOT, "profiles", tag + ".md"), "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        summarise_launches(sys.argv[2], sys.argv[3])
    else:
        tr = summarise_full(sys.argv[1], sys.argv[2])
        tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        cur = json.load(open(tj)) if os.path.exists(tj) else {}
        key = sys.argv[3] if len(sys.argv) > 3 else sys.argv[2]
        cur.setdefault(key, {}).update(tr)
        json.dump(cur, open(tj, "w"), indent=1)
