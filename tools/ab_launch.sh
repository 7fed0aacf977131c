#!/bin/bash
# A/B per-kernel warm launch lists: default build vs build_variants/$v
#   VARIANTS="a b" tools/ab_launch.sh c2 c4   -> gpurun_out/ab_<variant>_<config>.txt
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for v in default ${VARIANTS}; do
  if [ $v = default ]; then unset VF_LIB_PATH; else export VF_LIB_PATH=$PWD/build_variants/$v/libvoxforest_b200.so; fi
  for c in ${@:-c2 c4}; do
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
      --log-file gpurun_out/ab_${v}_$c.csv python tools/one_embed.py $c 2 > /dev/null 2>&1
    python tools/ncu_summary.py gpurun_out/ab_${v}_$c.csv 2 > gpurun_out/ab_${v}_$c.txt
  done
done
