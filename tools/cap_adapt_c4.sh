# source-level ncu capture of k_voxelize at the finest C4 level
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_adapt_children -s 3 -c 1 -o /tmp/vox4 -f python tools/one_embed.py c4 1 > gpurun_out/cap_vox.log 2>&1
python tools/ncu_lines.py /tmp/vox4.ncu-rep regex:k_adapt_children 30 > gpurun_out/vox4_lines.txt 2>&1
python tools/ncu_sass_hot.py /tmp/vox4.ncu-rep regex:k_adapt_children 20 > gpurun_out/vox4_sass.txt 2>&1
ncu -i /tmp/vox4.ncu-rep --page details --csv > gpurun_out/vox4_details.csv 2>&1
