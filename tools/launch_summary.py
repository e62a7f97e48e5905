"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, total, mean."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"][:70]
    agg.setdefault(k, []).append(float(d["Metric Value"]))
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    print(f"{k:70s} n={len(v):4d} total={sum(v) / 1e6:9.3f} ms mean={sum(v) / len(v) / 1e3:9.1f} us  {100 * sum(v) / tot:5.1f}%")
