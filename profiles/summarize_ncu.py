#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum CSV) and a --set full
report into a committed markdown file + a traffic JSON the bench reads.

usage: python profiles/summarize_ncu.py TAG CONFIG FORM [launches.csv] [prof.ncu-rep]

Writes profiles/r02/ncu/TAG_ncu_summary.md and, from the --set full report, the evidence file
profiles/r02/ncu/traffic_CONFIG_FORM.json (DRAM bytes, MUFU / issue / SM-clock figures of the
dominant kernel) stamped with bench.src_sha() of the sources it was captured on: bench.py uses
it as `roofline.traffic` only while the kernel sources are unchanged.
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
    tag, cfg, form = sys.argv[1], sys.argv[2], sys.argv[3]
    lpath = sys.argv[4] if len(sys.argv) > 4 else None
    ppath = sys.argv[5] if len(sys.argv) > 5 else None
    outdir = os.path.join(HERE, "r02", "ncu")
    os.makedirs(outdir, exist_ok=True)
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
                traffic.setdefault(d["kernel"].split("(")[0], []).append((rb + wb, d))
            md.append("")
    open(os.path.join(outdir, f"{tag}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    if traffic:
        sys.path.insert(0, os.path.dirname(HERE))
        import bench
        # the call's kernels (each captured once, e.g. the two-pass forward, pair reduction and
        # backward): traffic per call = their sum; the pipe figures are the dominant kernel's
        main_k = max(traffic, key=lambda k: sum(t for t, _ in traffic[k]) / len(traffic[k]))
        v = traffic[main_k]
        d = v[0][1]
        per_call = sum(sum(t for t, _ in vv) / len(vv) for vv in traffic.values())

        def num(key, scale=1.0):
            return float(d[key][0].replace(",", "")) * scale if key in d else None
        ev = {"kernel": " + ".join(traffic.keys()), "dominant_kernel": main_k,
              "dram_bytes_per_launch": per_call,
              "dram_read_bytes": to_bytes(*d["dram__bytes_read.sum"]),
              "dram_write_bytes": to_bytes(*d["dram__bytes_write.sum"]),
              "duration_ms": num("gpu__time_duration.sum") / 1e6
              if d.get("gpu__time_duration.sum", ("", ""))[1] == "nsecond"
              else num("gpu__time_duration.sum") if d.get("gpu__time_duration.sum", ("", ""))[1] == "msecond"
              else None,
              "mufu_pipe_pct": num("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
              "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
              "dram_pct_of_peak": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
              "l2_hit_pct": num("lts__t_sector_hit_rate.pct"),
              "sm_clock": " ".join(d.get("sm__cycles_elapsed.avg.per_second", ("", ""))),
              "tag": tag, "src_sha": bench.src_sha(),
              "how": "ncu --set full --clock-control none (one launch, cold cache)"}
        json.dump(ev, open(os.path.join(outdir, f"traffic_{cfg}_{form}.json"), "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
