#!/bin/bash
# A/B of enumeration build variants (build_variants/, tools/build_variant.sh):
# link parity tests under each variant, then tools/ab_quick.sh timings.
#   VARIANTS="p2 p4" tools/ab_enum.sh c4 c2
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for v in ${VARIANTS}; do
  echo "== parity $v"
  VF_LIB_PATH=$PWD/build_variants/$v/libvoxforest_b200.so timeout 600 python -m pytest -q -x -m gpu tests/test_gpu_parity.py \
    -k "small_face or c2_bench or c4_flagship or edges_small or grid_aligned or boundary_tables" 2>&1 | tail -1
done
KT_GREP="${KT_GREP:-k_links_small}" bash tools/ab_quick.sh "$@"
