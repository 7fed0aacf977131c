cd $GRAFT_REPO_ROOT
timeout 1200 ncu --set full --clock-control none -k regex:"k_links|k_voxelize|k_pairs|k_adapt_children|k_boundary|k_xrows|k_indicators_all|k_fill_lut" -s 40 -c 40 -o /tmp/full_c2 -f python tools/one_embed.py c2 2 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_traffic.py /tmp/full_c2.ncu-rep c2 > gpurun_out/ncu_traffic_c2.txt 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:"k_links|k_fill_lut" -s 5 -c 5 -o /tmp/full_c4 -f python tools/one_embed.py c4 2 > gpurun_out/ncu_full_c4.log 2>&1
python tools/ncu_traffic.py /tmp/full_c4.ncu-rep c4 > gpurun_out/ncu_traffic_c4.txt 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
cat gpurun_out/ncu_traffic_c2.txt gpurun_out/ncu_traffic_c4.txt
