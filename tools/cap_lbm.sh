# source-level ncu capture of the bulk collide/stream kernel (C3 level 0)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_lbm_cells" -s 4 -c 1 -o /tmp/lbm -f python tools/one_lbm.py > gpurun_out/cap_lbm.log 2>&1
python tools/ncu_lines.py /tmp/lbm.ncu-rep regex:k_lbm_cells 25 > gpurun_out/lbm_lines.txt 2>&1
python tools/ncu_sass_hot.py /tmp/lbm.ncu-rep regex:k_lbm_cells 12 > gpurun_out/lbm_sass.txt 2>&1
ncu -i /tmp/lbm.ncu-rep --page details --csv > gpurun_out/lbm_details.csv 2>&1
