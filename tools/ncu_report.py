"""Key metrics + stall breakdown + hottest SASS of one ncu report."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ("Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "DRAM Throughput", "Compute (SM) Throughput", "Executed Instructions",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Memory Throughput", "Block Limit Registers")
rows_d = list(csv.reader(det.splitlines()))
hd = rows_d[0]
mi, ui, vi = hd.index("Metric Name"), hd.index("Metric Unit"), hd.index("Metric Value")
for row in rows_d[1:]:
    if len(row) > vi and row[mi] in want:
        print(f"{row[mi]:28s} {row[vi]:>14s} {row[ui]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(src))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: sum(int(r[hdr.index(c)]) for r in data) for c in cols}
s = sum(tot.values()) or 1
print("stalls:", ", ".join(f"{c[6:]} {v / s * 100:.0f}%" for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:6]))
ws = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
tws = sum(int(r[ws]) for r in data) or 1
top = sorted(range(len(data)), key=lambda i: -int(data[i][ws]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]
for i in sorted(top):
    print(f"{i:5d} {data[i][1].strip()[:64]:64s} exec={data[i][ie]:>10s} stall={int(data[i][ws]) / tws * 100:5.1f}%")
print("sass lines", len(data))
