"""Per-CUDA-source-line totals (executed warp instructions, stall samples) of an ncu capture taken with
-lineinfo and --import-source on.  usage: python tools/ncu_line_summary.py <report.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True, check=True).stdout
    f = "?"
    tot = {}
    hdr = None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if not r[0]:
            continue   # SASS rows: the line row before them carries the line's totals
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        iI = hdr.index("Instructions Executed")
        a = tot.setdefault((f, int(r[0])), [0, 0, r[1]])
        a[0] += int(r[iI]) if r[iI].isdigit() else 0
        a[1] += int(r[iS]) if r[iS].isdigit() else 0
    ni = sum(v[0] for v in tot.values()) or 1
    ns = sum(v[1] for v in tot.values()) or 1
    print(f"| file:line | % inst | % samples | source |\n|---|---|---|---|")
    for (fn, ln), (i, s, src) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"| {fn}:{ln} | {i / ni:.1%} | {s / ns:.1%} | `{src.strip()[:70]}` |")


if __name__ == "__main__":
    main()
