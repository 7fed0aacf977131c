#!/bin/bash
# ncu --set full capture of selected kernels of a steady-state embed
#   tools/ncu_kernel.sh <c2|c4> <kernel regex> <skip> <count> <out name>
# report -> gpurun_out/<out>.ncu-rep (read here with ncu -i / tools/ncu_report.py)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"$2" -s "$3" -c "$4" \
  -o gpurun_out/$5 -f python tools/one_embed.py $1 2 > gpurun_out/$5.log 2>&1
