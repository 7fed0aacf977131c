# source-level ncu capture of the finest-level pipeline kernels at C2 (second
# embed): k_adapt_children (L2->L3), k_voxelize (L3), k_xrows (L3)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_xrows|k_voxelize|k_adapt_children" -s 19 -c 3 -o /tmp/lvl -f python tools/one_embed.py c2 2 > gpurun_out/cap_level.log 2>&1
for k in k_adapt_children k_voxelize k_xrows; do
  python tools/ncu_lines.py /tmp/lvl.ncu-rep regex:$k 25 > gpurun_out/lvl_${k}_lines.txt 2>&1
  python tools/ncu_sass_hot.py /tmp/lvl.ncu-rep regex:$k 12 > gpurun_out/lvl_${k}_sass.txt 2>&1
done
ncu -i /tmp/lvl.ncu-rep --page details --csv > gpurun_out/lvl_details.csv 2>&1
