"""Summarise ncu --set full captures (.ncu-rep) into a markdown table for profiles/: per kernel launch the
duration, DRAM bytes (read + write), issue-active, registers, occupancy and the top warp-stall reasons.
Usage: python tools/ncu_summary.py out.md rep1.ncu-rep [rep2 ...]"""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "smsp__inst_executed.sum": "warp_instr",
}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    h, units = r[0], r[1]
    res = []
    for v in r[2:]:
        d = {"kernel": v[h.index("Kernel Name")][:60] if "Kernel Name" in h else "?"}
        for k, name in KEYS.items():
            if k in h:
                i = h.index(k)
                d[name] = (v[i], units[i])
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(v[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        tot = sum(s for s, _ in stalls) or 1.0
        d["stalls"] = ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in stalls[:4])
        res.append(d)
    return res


def fmt(d, k):
    if k not in d:
        return "-"
    v, u = d[k]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    if k == "time":
        return {"usecond": f"{x / 1e3:.4f} ms", "msecond": f"{x:.4f} ms", "nsecond": f"{x / 1e6:.4f} ms"}.get(u, f"{x} {u}")
    if k in ("dram_rd", "dram_wr"):
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
        return f"{x * scale:.1f} MB"
    return f"{x:g}"


def main():
    out = sys.argv[1]
    lines = ["| capture | kernel | time | DRAM read | DRAM write | issue-active % | regs | warps active % | warp instr | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for rep in sys.argv[2:]:
        for d in rows(rep):
            lines.append(f"| {rep.split('/')[-1]} | `{d['kernel']}` | {fmt(d, 'time')} | {fmt(d, 'dram_rd')} | "
                         f"{fmt(d, 'dram_wr')} | {fmt(d, 'issue%')} | {fmt(d, 'regs')} | {fmt(d, 'occ%')} | "
                         f"{fmt(d, 'warp_instr')} | {d['stalls']} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
