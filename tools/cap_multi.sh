#!/bin/bash
# ncu --set full of several kernels of one steady-state embed: summary per kernel
#   tools/cap_multi.sh <c2|c4> <kernel regex> <count> <out name>
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"$2" -c "$3" -o /tmp/$4 -f python tools/one_embed.py $1 1 > gpurun_out/$4.log 2>&1
python tools/ncu_traffic.py /tmp/$4.ncu-rep $1 > gpurun_out/$4_traffic.txt 2>&1
for k in $(echo "$2" | tr '|' ' '); do
  python tools/ncu_lines.py /tmp/$4.ncu-rep regex:"$k" 25 > gpurun_out/$4_${k}_lines.txt 2>&1
done
