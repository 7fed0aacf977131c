"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list:
tools/launch_sum.py <launches.csv> [first-kernel-substring]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
seq = [(d["Kernel Name"], float(d["Metric Value"].replace(",", "")) / 1e3) for d in data
       if d["Metric Name"] == "gpu__time_duration.sum"]
if len(sys.argv) > 2:
    seq = seq[[i for i, (n, _) in enumerate(seq) if sys.argv[2] in n][0]:]
k = collections.defaultdict(list)
for n, t in seq:
    k[n.split("(")[0][:48]].append(t)
for n, v in sorted(k.items(), key=lambda x: -sum(x[1])):
    print(f"{n:50s} n={len(v):4d} sum={sum(v):9.1f}us mean={sum(v) / len(v):7.2f}us")
