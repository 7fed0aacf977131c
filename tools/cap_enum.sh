# source-level ncu capture of one cut-link enumeration kernel
# usage: bash tools/cap_enum.sh [kernel-regex] [config: c4|c2]
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
K=${1:-k_links_small}
C=${2:-c4}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$K" -c 1 -o /tmp/enum_$C -f python tools/one_embed.py $C 1 > gpurun_out/cap.log 2>&1
python tools/ncu_lines.py /tmp/enum_$C.ncu-rep regex:"$K" 70 > gpurun_out/enum_${C}_lines.txt 2>&1
python tools/ncu_sass_hot.py /tmp/enum_$C.ncu-rep regex:"$K" 40 > gpurun_out/enum_${C}_sass.txt 2>&1
ncu -i /tmp/enum_$C.ncu-rep --page details --csv > gpurun_out/enum_${C}_details.csv 2>&1
