"""Summarise an ncu --csv launch list: mean time / dram bytes per kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(lambda: defaultdict(list))
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"])
        agg[key][d["Metric Name"]].append((float(d["Metric Value"].replace(",", "")), d["Metric Unit"]))
per = defaultdict(lambda: defaultdict(list))
for (i, name), m in agg.items():
    for k, v in m.items():
        per[name][k].append(v[0])
for name, m in per.items():
    if "camx" not in name and len(sys.argv) < 3:
        continue
    s = "  ".join(f"{k.split('__')[1]}={sum(x for x, _ in v)/len(v):.4g}{v[0][1]}" for k, v in m.items())
    print(f"{name[:50]:50s} n={len(next(iter(m.values())))} {s}")
