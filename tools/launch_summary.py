#!/usr/bin/env python3
"""Summarise an ncu --csv launch list (gpu__time_duration.sum + dram bytes per
launch) into a markdown table for profiles/: launches, mean duration, mean DRAM
read, share of the captured time per kernel.

Usage: python tools/launch_summary.py launches.csv "title" "command" > profiles/x.md
"""
import csv
import sys
from collections import defaultdict


def main(path, title, cmd):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    agg = defaultdict(lambda: defaultdict(list))
    scale = {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "byte": 1, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "")
        agg[name][r[12]].append(float(r[14].replace(",", "")) * scale.get(r[13], 1))
    total = sum(sum(m["gpu__time_duration.sum"]) for m in agg.values())
    print(f"# {title}\n\nCommand: `{cmd}` (cold caches, serialised: compare shares, not absolutes).\n")
    print("| kernel | launches | mean us | mean DRAM read MB | share of captured time |")
    print("|---|---|---|---|---|")
    for name, m in sorted(agg.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
        t = m["gpu__time_duration.sum"]
        rd = m.get("dram__bytes_read.sum", [])
        print(f"| {name} | {len(t)} | {sum(t) / len(t) / 1e3:.2f} | "
              f"{(sum(rd) / len(rd) / 1e6) if rd else float('nan'):.2f} | {sum(t) / total:.3f} |")


if __name__ == "__main__":
    main(*sys.argv[1:4])
