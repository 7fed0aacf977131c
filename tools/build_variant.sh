#!/bin/bash
# build_variant.sh NAME "NVCC -D flags": an alternative build of the library in
# build_variants/NAME/ for A/B timing (select with VF_LIB_PATH=...).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OUT=$ROOT/build_variants/$NAME
mkdir -p $OUT/obj
cd $ROOT/paper_2512_01251_b200/csrc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -ccbin /usr/bin/g++ $*"
for f in vf_api vf_bins vf_voxelize vf_forest vf_links vf_linklen vf_shard vf_lbm vf_stl vf_io vf_rows; do
  fm=-fmad=false; [ $f = vf_lbm ] && fm=-fmad=true
  /usr/local/cuda/bin/nvcc $FL $fm -c $f.cu -o $OUT/obj/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -o $OUT/libvoxforest_b200.so $OUT/obj/*.o -lcudart -lnccl
echo $OUT/libvoxforest_b200.so
