#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (committed evidence).

  python scripts/ncu_summary.py gpurun_out/prof_exchange.ncu-rep gpurun_out/launches.csv \
      --out profiles/r01_exchange.md --traffic-key one_peer_fp32_n1

Reads the raw page of a `--set full` report (per-kernel metrics) and the CSV
launch list of the `gpu__time_duration.sum` pass; writes a markdown summary and
updates profiles/traffic.json (DRAM bytes per launch, read by bench.py).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__maximum_warps_per_active_cycle_pct",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "nvlrx__bytes.sum", "nvltx__bytes.sum",
]


def raw_page(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for key in ["Kernel Name"] + KEYS:
            if key in hdr:
                i = hdr.index(key)
                d[key] = (r[i], units[i] if key != "Kernel Name" else "")
        res.append(d)
    return res


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return v * mult


def launches(path):
    shares = defaultdict(float)
    counts = defaultdict(int)
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        name = r[ki].split("(")[0].replace("void ", "")
        shares[name] += ns
        counts[name] += 1
    return shares, counts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("launch_csv", nargs="?")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic-key")
    ap.add_argument("--title", default="exchange_kernel")
    a = ap.parse_args()
    kern = raw_page(a.rep)
    lines = [f"# ncu summary: {a.title}", "", f"source: `{os.path.basename(a.rep)}` (`--set full --clock-control none`)", ""]
    traffic = None
    for d in kern:
        lines.append(f"## {d.get('Kernel Name', ('?',))[0][:120]}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for key in KEYS:
            if key in d:
                lines.append(f"| {key} | {d[key][0]} | {d[key][1]} |")
        if "dram__bytes_read.sum" in d:
            rb = to_bytes(*d["dram__bytes_read.sum"])
            wb = to_bytes(*d["dram__bytes_write.sum"])
            traffic = rb + wb
            lines.append(f"| dram read+write | {traffic / 1e9:.4f} | GB per launch |")
        lines.append("")
    if a.launch_csv and os.path.exists(a.launch_csv):
        shares, counts = launches(a.launch_csv)
        tot = sum(shares.values())
        lines += ["## launch list (gpu__time_duration.sum, cold-cache, serialised)", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for name, ns in sorted(shares.items(), key=lambda kv: -kv[1]):
            lines.append(f"| {name} | {counts[name]} | {ns / 1e6:.3f} | {ns / tot:.1%} |")
        lines.append("")
    with open(a.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if a.traffic_key and traffic is not None:
        tp = os.path.join(os.path.dirname(a.out), "traffic.json")
        tj = json.load(open(tp)) if os.path.exists(tp) else {}
        tj[a.traffic_key] = traffic
        json.dump(tj, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
