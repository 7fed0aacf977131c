cd $GRAFT_REPO_ROOT
for v in default minb6; do
  if [ $v = default ]; then unset VF_LIB_PATH; else export VF_LIB_PATH=$PWD/build_variants/$v/libvoxforest_b200.so; fi
  echo "== $v"; timeout 300 python tools/quick_embed.py c2 c4 2>&1 | sed 's/eager.*(k_links/(k_links/'
done
