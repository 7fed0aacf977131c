"""Group an ncu source-page (cuda,sass) profile of one kernel by enclosing
source function: stall samples, warp instructions, thread instructions.
usage: ncu_funcs.py <rep> <kernel> <source.cu>"""
import re, subprocess, sys
from collections import defaultdict
rep, kern, src = sys.argv[1:4]
out = subprocess.run([sys.executable, __file__.replace("ncu_funcs.py", "ncu_lines.py"), rep, kern, "100000"],
                     capture_output=True, text=True).stdout
lines = open(src).read().split("\n")
heads = []
for i, l in enumerate(lines, 1):
    if re.match(r"^(__device__|__global__|template|static|int |size_t )", l) or re.match(r"^    k_\w+\(", l):
        nm = re.findall(r"(\w+)\(", l)
        if nm:
            heads.append((i, nm[0]))
base = src.split("/")[-1]
agg = defaultdict(lambda: [0.0, 0.0, 0.0])
print(out.split("\n")[0])
for l in out.split("\n")[1:]:
    m = re.match(r"\s*([\d.]+)% st\s+([\d.]+)% wi\s+([\d.]+)% ti\s+(\S+):(\d+)", l)
    if not m:
        continue
    f, ln = m.group(4), int(m.group(5))
    key = f
    if f == base:
        key = "?"
        for i, n in heads:
            if i <= ln:
                key = n
    a = agg[key]
    for k in range(3):
        a[k] += float(m.group(k + 1))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:28s} stall {v[0]:5.1f}%  warp-inst {v[1]:5.1f}%  thread-inst {v[2]:5.1f}%")
