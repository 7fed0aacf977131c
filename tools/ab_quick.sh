#!/bin/bash
# A/B embed timings (tools/quick_embed.py, graph replay) and per-launch vox
# times: default build vs build_variants/$v.  VARIANTS="a b" tools/ab_quick.sh c4
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for rep in 1 2; do
for v in default ${VARIANTS}; do
  if [ $v = default ]; then unset VF_LIB_PATH; else export VF_LIB_PATH=$PWD/build_variants/$v/libvoxforest_b200.so; fi
  echo "== $v"; timeout 600 python tools/quick_embed.py ${@:-c4} 2>&1 | tail -3
  [ $rep = 1 ] && timeout 600 python tools/kt_each.py ${1:-c4} 2>&1 | grep -E "${KT_GREP:-k_voxelize}" | tr '\n' ' '; echo
done
done
