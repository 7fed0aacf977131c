"""Record per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
and the main throughput counters of the kernels in an ncu --set full report
into profiles/ncu_traffic.json under a workload key (bench.py reads it for the
roofline `traffic` field).

usage: python tools/ncu_traffic.py <report.ncu-rep> <workload key, e.g. c2>"""
import csv, io, json, os, re, subprocess, sys

rep, key = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
MB = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
US = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def val(row, name, scale=None):
    i = h.index(name)
    v = float(row[i].replace(",", ""))
    if scale is not None:
        v *= scale.get(units[i], 1.0)
    return v


res = {}
for row in rows[2:]:
    name = re.sub(r"\(.*", "", row[h.index("Kernel Name")]).replace("void ", "").strip()
    name = re.sub(r"^vf::", "", name)
    if name.startswith("k_links<"):  # MODE 0 direct / 1 overflow fallback / 2 line enumeration
        name = {"0": "k_links", "1": "k_links_full", "2": "k_links_enum"}.get(name[8:9], name)
    name = re.sub(r"<.*", "", name)
    d = {"launches": 1,
         "time_us": val(row, "gpu__time_duration.sum", US),
         "dram_bytes": val(row, "dram__bytes_read.sum", MB) + val(row, "dram__bytes_write.sum", MB),
         "dram_read_bytes": val(row, "dram__bytes_read.sum", MB),
         "dram_write_bytes": val(row, "dram__bytes_write.sum", MB),
         "sm_throughput_pct": val(row, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
         "dram_throughput_pct": val(row, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
         "warps_active_pct": val(row, "sm__warps_active.avg.pct_of_peak_sustained_active"),
         "registers": val(row, "launch__registers_per_thread"),
         "fp64_pipe_pct": val(row, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
         "threads_per_inst": val(row, "smsp__thread_inst_executed_per_inst_executed.ratio")}
    if name in res:  # several launches: keep the per-launch mean of additive fields
        a = res[name]
        n = a["launches"] + 1
        for k in d:
            if k != "launches":
                a[k] = (a[k] * a["launches"] + d[k]) / n
        a["launches"] = n
    else:
        res[name] = d
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
allv = json.load(open(path)) if os.path.exists(path) else {}
allv[key] = {"source": os.path.basename(rep), "kernels": res, **{k: v for k, v in res.items()}}
json.dump(allv, open(path, "w"), indent=1, sort_keys=True)
for k, v in sorted(res.items(), key=lambda kv: -kv[1]["time_us"]):
    print(f"{k:28s} n={v['launches']:3d} {v['time_us']:9.1f} us  dram {v['dram_bytes']/1e6:8.2f} MB  "
          f"sm {v['sm_throughput_pct']:5.1f}%  dram {v['dram_throughput_pct']:5.1f}%  warps {v['warps_active_pct']:5.1f}%")
