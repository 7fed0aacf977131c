"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel count, total and share of device time (per run if --runs N)."""
import csv, sys, collections, re
path = sys.argv[1]
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rows = list(csv.reader(open(path)))
hdr = None
data = []
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            data.append(d)
agg = collections.OrderedDict()
unit = data[0].get("Metric Unit", "") if data else ""
for d in data:
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")
    name = re.sub(r"<.*>", "<>", name)
    v = float(d["Metric Value"].replace(",", ""))
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
scale = 1e-3 if unit in ("nsecond", "ns") else (1.0 if unit in ("usecond", "us") else 1e-3)
print(f"launches={len(data)} total={tot*scale/runs:.1f} us/run (unit {unit}, runs={runs})")
for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v/tot*100:6.2f}%  {v*scale/runs:10.1f} us/run  {n/runs:7.1f} launches/run  {k}")
