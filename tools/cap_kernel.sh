#!/bin/bash
# ncu --set full capture of one launch of a kernel in a steady-state embed, summarised on the box
#   tools/cap_kernel.sh <c2|c4> <kernel regex> <skip> <out name>
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$2" -s "$3" -c 1 -o /tmp/$4 -f python tools/one_embed.py $1 ${NEMB:-2} > gpurun_out/$4.log 2>&1
python tools/ncu_lines.py /tmp/$4.ncu-rep regex:"$2" 40 > gpurun_out/$4_lines.txt 2>&1
python tools/ncu_sass_hot.py /tmp/$4.ncu-rep regex:"$2" 25 > gpurun_out/$4_sass.txt 2>&1
ncu -i /tmp/$4.ncu-rep --page details --csv > gpurun_out/$4_details.csv 2>&1
python tools/ncu_details.py gpurun_out/$4_details.csv > gpurun_out/$4_summary.txt 2>&1
