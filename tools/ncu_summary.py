#!/usr/bin/env python3
"""Summarise an ncu --set full report into markdown for profiles/.

Usage: python tools/ncu_summary.py report.ncu-rep "title" [algorithmic_bytes] > profiles/x.md
Prints duration, DRAM bytes read/written (traffic), achieved DRAM GB/s, SM /
DRAM throughput %, occupancy, registers, the warp-state headline and the top
source lines by stall samples (needs -lineinfo builds).
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__inst_executed.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k, u, v in zip(hdr, units, r):
            d[k] = (v, u)
        res.append(d)
    return res


def main():
    rep, title = sys.argv[1], sys.argv[2]
    alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
    for d in raw(rep):
        name = d.get("Kernel Name", ("?", ""))[0]
        print(f"# {title}\n\nKernel: `{name[:120]}`  (report `{rep.split('/')[-1]}`)\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in d:
                print(f"| {k} | {d[k][0]} | {d[k][1]} |")
        try:
            t = float(d["gpu__time_duration.sum"][0].replace(",", ""))
            tu = d["gpu__time_duration.sum"][1]
            ts = t * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(tu, 1e-9)
            rb = float(d["dram__bytes_read.sum"][0].replace(",", ""))
            wb = float(d["dram__bytes_write.sum"][0].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rb *= scale.get(d["dram__bytes_read.sum"][1], 1)
            wb *= scale.get(d["dram__bytes_write.sum"][1], 1)
            print(f"\nDRAM traffic per launch: {(rb + wb) / 1e6:.2f} MB (read {rb / 1e6:.2f}, write {wb / 1e6:.2f}); "
                  f"achieved {(rb + wb) / ts / 1e9:.0f} GB/s over {ts * 1e6:.2f} us (ncu: cold caches, serialised).")
            if alg:
                print(f"Algorithmic bytes per launch: {alg / 1e6:.2f} MB -> traffic / algorithmic = {(rb + wb) / alg:.3f}.")
        except Exception as e:  # noqa: BLE001
            print(f"(traffic unavailable: {e})")
    src = subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_hot.py"), rep, "15"],
                         capture_output=True, text=True).stdout
    print("\nTop source lines by warp-stall samples:\n\n```\n" + src.strip() + "\n```")


if __name__ == "__main__":
    main()
