#!/bin/bash
# ncu --set full of k_lbm_special at level 1 and level 2 of the C3 probe
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
tag=${1:-sp}
for k in ${KS:-15 28}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_lbm_special -s $k -c 1 \
    -o /tmp/${tag}_$k -f python tools/lbm_probe.py 2 > gpurun_out/${tag}_$k.log 2>&1
  ncu -i /tmp/${tag}_$k.ncu-rep --page details --csv > gpurun_out/${tag}_${k}_details.csv 2>&1
  python tools/ncu_details.py gpurun_out/${tag}_${k}_details.csv > gpurun_out/${tag}_${k}_summary.txt 2>&1
  python tools/ncu_lines.py /tmp/${tag}_$k.ncu-rep regex:k_lbm_special 30 > gpurun_out/${tag}_${k}_lines.txt 2>&1
done
