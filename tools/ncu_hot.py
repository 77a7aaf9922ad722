#!/usr/bin/env python3
"""Summarise an ncu report's warp-stall samples per CUDA source line.

Usage: python tools/ncu_hot.py report.ncu-rep [top]
Reads `ncu -i <rep> --page source --csv --print-source cuda,sass` and sums the
SASS-level "Warp Stall Sampling (All Samples)" of each instruction into the
CUDA line it belongs to.
"""
import csv
import subprocess
import sys
from collections import defaultdict


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    agg = defaultdict(int)
    src = {}
    path, cur, hdr = None, None, None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        if r[0] == "Function Name":
            continue
        if r[0]:
            if not r[0].isdigit():
                continue
            cur = (path, int(r[0]))
            src[cur] = r[1].strip()[:100]
        try:
            s = int(r[4] or 0)
        except (ValueError, IndexError):
            continue
        if cur:
            agg[cur] += s
    tot = sum(agg.values()) or 1
    print(f"total samples {tot}")
    for k, s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100.0 * s / tot:5.1f}% {k[0]}:{k[1]}  {src.get(k, '')}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
