"""Summarise the SASS source page of an ncu capture (--import-source on): stall-reason totals, the hottest
instructions by executed warp instructions and by stall samples, and optional address regions.

usage: python tools/ncu_source_summary.py <report.ncu-rep> [lo:hi:name ...]   (hex offsets, low 20 bits)
"""
import csv
import io
import subprocess
import sys


def main():
    rep, *regions = sys.argv[1:]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    ci = {c: hdr.index(c) for c in cols}
    ii = hdr.index("Instructions Executed")
    data = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        data.append((int(r[0], 16) & 0xFFFFF, r[1].strip(), int(r[ii] or 0), {c: int(r[ci[c]] or 0) for c in cols}))
    ninst = sum(d[2] for d in data)
    tot = {c: sum(d[3][c] for d in data) for c in cols}
    nsmp = sum(tot.values())
    print(f"# {rep}\n\nexecuted warp instructions: {ninst:,}; stall samples: {nsmp:,}\n")
    print("| stall reason | share of samples |\n|---|---|")
    for c, v in sorted(tot.items(), key=lambda x: -x[1]):
        if v > 0.005 * nsmp:
            print(f"| {c[6:]} | {v / nsmp:.1%} |")
    print("\n## hottest instructions (executed)\n\n| offset | % inst | % samples | SASS |\n|---|---|---|---|")
    for a, s, n, st in sorted(data, key=lambda d: -d[2])[:25]:
        print(f"| {a:05x} | {n / ninst:.2%} | {sum(st.values()) / nsmp:.2%} | `{s[:70]}` |")
    print("\n## hottest instructions (stall samples)\n\n| offset | % samples | top reason | SASS |\n|---|---|---|---|")
    for a, s, n, st in sorted(data, key=lambda d: -sum(d[3].values()))[:20]:
        top = max(st, key=st.get)
        print(f"| {a:05x} | {sum(st.values()) / nsmp:.2%} | {top[6:]} | `{s[:70]}` |")
    if regions:
        print("\n## regions\n\n| region | % inst | % samples | top reasons |\n|---|---|---|---|")
        for spec in regions:
            lo, hi, name = spec.split(":")
            lo, hi = int(lo, 16), int(hi, 16)
            sel = [d for d in data if lo <= d[0] < hi]
            n = sum(d[2] for d in sel)
            rt = {c: sum(d[3][c] for d in sel) for c in cols}
            sm = sum(rt.values())
            top = ", ".join(f"{c[6:]} {v / max(sm, 1):.0%}" for c, v in sorted(rt.items(), key=lambda x: -x[1])[:5])
            print(f"| {name} | {n / ninst:.1%} | {sm / nsmp:.1%} | {top} |")


if __name__ == "__main__":
    main()
