#!/bin/bash
# LBM probe on the box: timings, launch list, ncu --set full of the bulk
# collide/stream and the ghost fill
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
tag=${1:-lbm}
python tools/lbm_probe.py 10 > gpurun_out/${tag}_probe.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/${tag}_launches.csv python tools/lbm_probe.py 2 > /dev/null 2>&1
for k in "k_lbm_bulk:8" "k_lbm_special:8" "k_lbm_fill_ghosts:4" "k_lbm_restrict:2"; do
  name=${k%%:*}; skip=${k##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$name" -s $skip -c 1 \
    -o /tmp/${tag}_$name -f python tools/lbm_probe.py 2 > gpurun_out/${tag}_${name}.log 2>&1
  ncu -i /tmp/${tag}_$name.ncu-rep --page details --csv > gpurun_out/${tag}_${name}_details.csv 2>&1
  python tools/ncu_details.py gpurun_out/${tag}_${name}_details.csv > gpurun_out/${tag}_${name}_summary.txt 2>&1
  python tools/ncu_lines.py /tmp/${tag}_$name.ncu-rep regex:"$name" 30 > gpurun_out/${tag}_${name}_lines.txt 2>&1
done
