#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum CSV) and a --set full
report into a committed markdown file + a traffic JSON the bench reads.

usage: python profiles/summarize_ncu.py TAG CONFIG [launches.csv] [prof.ncu-rep]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict

HERE = os.path.dirname(os.path.abspath(__file__))

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def to_bytes(val, unit):
    v = float(val)
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return v * mult


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: j for j, h in enumerate(hdr)}
    agg = OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0]
        agg.setdefault(name, []).append(float(r[ix["Metric Value"]].replace(",", "")))
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, _ in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (r[i], units[i])
        res.append(d)
    return res


def main():
    tag, cfg = sys.argv[1], sys.argv[2]
    lpath = sys.argv[3] if len(sys.argv) > 3 else None
    ppath = sys.argv[4] if len(sys.argv) > 4 else None
    md = [f"# ncu summary {tag} ({cfg})", ""]
    if lpath and os.path.exists(lpath):
        agg = launches(lpath)
        tot = sum(sum(v) for v in agg.values())
        md += ["## launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
               "", "| kernel | launches | mean us | share of listed time |", "|---|---|---|---|"]
        for k, v in agg.items():
            md.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
        md.append("")
    traffic = {}
    if ppath and os.path.exists(ppath):
        md += ["## --set full (per launch)", ""]
        for d in full(ppath):
            md.append(f"### `{d['kernel']}`")
            for k, label in KEYS:
                if k in d:
                    md.append(f"- {label} (`{k}`): {d[k][0]} {d[k][1]}")
            if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d:
                rb = to_bytes(*d["dram__bytes_read.sum"])
                wb = to_bytes(*d["dram__bytes_write.sum"])
                md.append(f"- DRAM traffic per launch: {(rb + wb) / 1e9:.3f} GB")
                traffic.setdefault(d["kernel"].split("(")[0], []).append(rb + wb)
            md.append("")
    open(os.path.join(HERE, f"{tag}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    if traffic:
        main_k = max(traffic, key=lambda k: sum(traffic[k]) / len(traffic[k]))
        v = traffic[main_k]
        json.dump({"kernel": main_k, "dram_bytes_per_launch": sum(v) / len(v), "tag": tag},
                  open(os.path.join(HERE, f"ncu_traffic_{cfg}.json"), "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
