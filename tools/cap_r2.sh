# source-level ncu captures of the C4 hot kernels (enumeration, voxelize finest level, resolve)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
bash tools/cap_enum.sh k_links_small c4
bash tools/cap_vox_c4.sh
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_links_resolve|k_fill_lut|k_indicators_all|k_adapt_children" -c 6 -o /tmp/res4 -f python tools/one_embed.py c4 1 > gpurun_out/cap_res.log 2>&1
python tools/ncu_traffic.py /tmp/res4.ncu-rep c4 > gpurun_out/res4_traffic.txt 2>&1
python tools/ncu_lines.py /tmp/res4.ncu-rep regex:k_links_resolve 30 > gpurun_out/res4_lines.txt 2>&1
python tools/ncu_lines.py /tmp/res4.ncu-rep regex:k_indicators_all 40 > gpurun_out/ind4_lines.txt 2>&1
ls -la gpurun_out
