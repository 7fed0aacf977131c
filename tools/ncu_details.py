"""Key metrics of an ncu --page details --csv export: usage ncu_details.py <csv>"""
import csv, sys
keys = ('Duration', 'Compute (SM) Throughput', 'Memory Throughput', 'DRAM Throughput', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Issue Slots Busy', 'Executed Ipc Active',
        'Avg. Active Threads Per Warp', 'No Eligible', 'Warp Cycles Per Issued Instruction',
        'Executed Instructions', 'Block Limit Registers', 'Block Limit Shared Mem', 'L2 Hit Rate', 'L1/TEX Hit Rate')
rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
seen = set()
for r in rows[1:]:
    d = dict(zip(h, r))
    k = d.get('Metric Name')
    if k in keys and k not in seen:
        seen.add(k)
        print(f"{k:40s} {d['Metric Value']} {d.get('Metric Unit', '')}")
