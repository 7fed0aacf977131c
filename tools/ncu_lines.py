"""Per-source-line stall samples / executed instructions of one kernel from an
ncu report (needs -lineinfo).  usage: ncu_lines.py <rep> <kernel> [top] [launch skip]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern,
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, fname, h = [], None, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = r
        continue
    if h is None or len(r) < 9 or not r[0]:
        continue
    try:
        res.append((int(float(r[4] or 0)), int(float(r[7] or 0)), int(float(r[8] or 0)), fname, r[0], r[1].strip()[:90]))
    except ValueError:
        pass
ts = sum(x[0] for x in res) or 1
ti = sum(x[1] for x in res) or 1
tt = sum(x[2] for x in res) or 1
print(f"stall samples {ts}, warp inst {ti}, thread inst {tt}")
for x in sorted(res, reverse=True)[:top]:
    print(f"{100*x[0]/ts:5.1f}% st {100*x[1]/ti:5.1f}% wi {100*x[2]/tt:5.1f}% ti  {x[3]}:{x[4]}  {x[5]}")
