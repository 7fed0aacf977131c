# source-level ncu capture of one cut-link enumeration kernel at C4
# usage: bash tools/cap_enum.sh [kernel-regex]
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
K=${1:-k_links_small}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$K" -c 1 -o /tmp/enum_c4 -f python tools/one_embed.py c4 1 > gpurun_out/cap.log 2>&1
python tools/ncu_lines.py /tmp/enum_c4.ncu-rep regex:$K 70 > gpurun_out/enum_c4_lines.txt 2>&1
python tools/ncu_sass_hot.py /tmp/enum_c4.ncu-rep regex:$K 40 > gpurun_out/enum_c4_sass.txt 2>&1
ncu -i /tmp/enum_c4.ncu-rep --page details --csv > gpurun_out/enum_c4_details.csv 2>&1
