"""Markdown tables for a round's profiles/<tag>/README.md from the gpurun_out/ files of
tools/round_profile.sh: the bench lines (one row per JSON file) and, per `ncu --set full`
capture, each kernel's duration, DRAM bytes and achieved bandwidth.

usage: python tools/profile_tables.py <tag> [gpurun_out]
"""
import csv
import glob
import json
import os
import subprocess
import sys


def bench_rows(tag, d):
    out = ["| file | value | unit | ms / step | e2e | roofline frac | k_inner / kernel | clocks (MHz, reasons) |",
           "|---|---|---|---|---|---|---|---|"]
    for p in sorted(glob.glob(os.path.join(d, f"{tag}_bench_*.json"))):
        try:
            j = json.loads(open(p).read().strip().splitlines()[-1])
        except Exception:
            continue
        r = j.get("roofline") or {}
        e2e = j.get("e2e") or {}
        clk = j.get("clocks") or {}
        out.append(f"| {os.path.basename(p)[len(tag) + 7:-5]} | {j.get('value'):,} | {j.get('unit')} | "
                   f"{j.get('ms_per_step')} | {e2e.get('value', '')} | {r.get('frac', '')} | "
                   f"{r.get('k_inner', r.get('kernel', ''))} | {clk.get('sm_mhz', '')}, {clk.get('reasons', '')} |")
    return "\n".join(out)


def traffic_rows(tag, d):
    out = ["| capture | kernel | duration ms | DRAM read MB | DRAM write MB | GB/s |", "|---|---|---|---|---|---|"]
    for p in sorted(glob.glob(os.path.join(d, f"{tag}_prof_*.ncu-rep"))):
        txt = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(txt.splitlines()))
        if len(rows) < 3:
            continue
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            v = dict(zip(h, r))
            u = dict(zip(h, units))

            def num(k, scale_to):
                x = float(v.get(k, "0").replace(",", "") or 0)
                unit = u.get(k, "")
                f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1, "s": 1e3,
                     "usecond": 1e-3, "msecond": 1, "nsecond": 1e-6}.get(unit, 1)
                return x * f / scale_to

            ms = num("gpu__time_duration.sum", 1)
            rd = num("dram__bytes_read.sum", 1e6)
            wr = num("dram__bytes_write.sum", 1e6)
            name = v.get("Kernel Name", "").split("(")[0].replace("fcfs::", "").replace("tc::", "").replace("fr::", "")
            bw = (rd + wr) / ms if ms > 0 else 0.0
            out.append(f"| {os.path.basename(p)[len(tag) + 6:-8]} | `{name[:60]}` | {ms:.3f} | {rd:.1f} | {wr:.1f} | "
                       f"{bw:.0f} |")
    return "\n".join(out)


if __name__ == "__main__":
    tag = sys.argv[1]
    d = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
    print("Bench lines:\n")
    print(bench_rows(tag, d))
    print("\nPer-kernel DRAM traffic (`ncu --set full`, one launch each):\n")
    print(traffic_rows(tag, d))
