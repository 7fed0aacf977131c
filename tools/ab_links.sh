# A/B: default build vs build_variants/$V (VARIANTS="a b")
cd $GRAFT_REPO_ROOT
for v in default ${VARIANTS}; do
  if [ $v = default ]; then unset VF_LIB_PATH; else export VF_LIB_PATH=$PWD/build_variants/$v/libvoxforest_b200.so; fi
  echo "== $v"; timeout 300 python tools/quick_embed.py c1 c2 c4 2>&1 | sed 's/eager=[0-9.]*ms //'
done
