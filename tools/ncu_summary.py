"""Summarise ncu outputs into a markdown file under profiles/.

usage: python tools/ncu_summary.py --launches gpurun_out/launches.csv --rep gpurun_out/prof.ncu-rep \
           --bench gpurun_out/bench.log --out profiles/r01_summary.md
"""
import argparse
import collections
import csv
import json
import subprocess

RAW_KEYS = [
    "gpu__time_duration.sum",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__warps_eligible.avg.per_cycle_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__bytes.sum.per_second",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__cycles_elapsed.avg",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    idx = {k: i for i, k in enumerate(h)}
    agg = collections.defaultdict(list)
    unit = ""
    for r in rows[1:]:
        if r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        unit = r[idx["Metric Unit"]] if "Metric Unit" in idx else unit
        agg[r[idx["Kernel Name"]].split("(")[0]].append(float(r[idx["Metric Value"]]))
    scale = 1e-3 if unit == "ns" else (1.0 if unit == "us" else 1e3)
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) * scale:.1f} | {sum(v) / tot:.1%} |")
    return "\n".join(out)


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    out = []
    for r in rows[2:]:
        d = dict(zip(rows[0], r))
        name = d.get("Kernel Name", "")[:80]
        out.append(f"\n**{name}**\n")
        out.append("| metric | value |\n|---|---|")
        for k in RAW_KEYS:
            if k in d:
                out.append(f"| `{k}` | {d[k]} |")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--bench")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    a = ap.parse_args()
    parts = [f"# {a.title}\n"]
    if a.bench:
        line = open(a.bench).read().strip().splitlines()[-1]
        d = json.loads(line)
        parts.append("## bench line (no profiler)\n\n```json\n" + json.dumps(d, indent=1) + "\n```\n")
    if a.launches:
        parts.append("## launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, "
                     "serialised: compare shares)\n\n" + launches(a.launches) + "\n")
    for rep in a.rep:
        parts.append(f"## ncu --set full: `{rep}`\n" + raw(rep) + "\n")
    open(a.out, "w").write("\n".join(parts))
    print(a.out)


if __name__ == "__main__":
    main()
