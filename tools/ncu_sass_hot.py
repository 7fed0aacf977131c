"""Summarise an ncu source page (SASS) CSV: stall samples and executed
instructions by opcode, plus the hottest address windows.
usage: python tools/ncu_sass_hot.py <report.ncu-rep> <kernel-regex> [top]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
A, S, W, I = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
data = []
for r in rows[hi + 1:]:
    if len(r) < len(h) or not r[A].startswith("0x"):
        continue
    data.append((int(r[A], 16), r[S].strip(), int(float(r[W] or 0)), int(float(r[I] or 0)),
                 {c: int(float(r[h.index(c)] or 0)) for c in stalls}))
ts = sum(d[2] for d in data) or 1
ti = sum(d[3] for d in data) or 1
print(f"{len(data)} SASS instructions, {ts} stall samples, {ti} warp-instructions executed")
op_s, op_i = defaultdict(int), defaultdict(int)
for d in data:
    op = d[1].split()[0] if not d[1].startswith("@") else d[1].split()[1]
    op = op.split(".")[0]
    op_s[op] += d[2]; op_i[op] += d[3]
print("by opcode (stall% / inst%):")
for op in sorted(op_s, key=lambda o: -op_s[o])[:top]:
    print(f"  {op:10s} {100*op_s[op]/ts:5.1f}% {100*op_i[op]/ti:5.1f}%")
agg = defaultdict(int)
for d in data:
    for c, v in d[4].items():
        agg[c] += v
print("stall reasons:", ", ".join(f"{c[6:]}={100*v/ts:.1f}%" for c, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
base = data[0][0]
win = defaultdict(lambda: [0, 0])
for d in data:
    k = (d[0] - base) // (16 * 32)
    win[k][0] += d[2]; win[k][1] += d[3]
print("hottest 32-instruction windows (offset: stall% inst%):")
for k in sorted(win, key=lambda k: -win[k][0])[:12]:
    print(f"  +0x{k*512:05x}: {100*win[k][0]/ts:5.1f}% {100*win[k][1]/ti:5.1f}%")
