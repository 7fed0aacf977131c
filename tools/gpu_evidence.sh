#!/bin/bash
# Round evidence on one B200: bench lines (C2 default, C4), ncu launch lists
# (C2, C4) and an ncu --set full capture of the dominant kernels at C2,
# summarised on the box (reports stay in /tmp; only summaries come back).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config c4 --steps 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
timeout 600 python tools/bench_stl.py c2 > gpurun_out/bench_stl_c2.json 2> gpurun_out/bench_stl_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/one_embed.py c2 3 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/one_embed.py c4 2 > /dev/null 2>&1
# steady-state launches: skip the first embed of one_embed (phase1 + phase2 eager)
timeout 1200 ncu --set full --clock-control none -k regex:"k_links|k_voxelize|k_pairs|k_adapt_children|k_boundary|k_xrows|k_indicators_all|k_fill_lut" -s 40 -c 40 -o /tmp/full_c2 -f python tools/one_embed.py c2 2 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_traffic.py /tmp/full_c2.ncu-rep c2 > gpurun_out/ncu_traffic_c2.txt 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:"k_links|k_fill_lut" -s 5 -c 5 -o /tmp/full_c4 -f python tools/one_embed.py c4 2 > gpurun_out/ncu_full_c4.log 2>&1
python tools/ncu_traffic.py /tmp/full_c4.ncu-rep c4 > gpurun_out/ncu_traffic_c4.txt 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
python tools/ncu_summary.py gpurun_out/launches_c2.csv 3 > gpurun_out/launches_c2.txt
python tools/ncu_summary.py gpurun_out/launches_c4.csv 2 > gpurun_out/launches_c4.txt
cat gpurun_out/bench_c2.json gpurun_out/ncu_traffic_c2.txt
# warm-cache launch lists (shares without ncu's per-kernel cache flush)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/warm_c2.csv python tools/one_embed.py c2 3 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/warm_c4.csv python tools/one_embed.py c4 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/warm_c2.csv 3 > gpurun_out/warm_c2.txt
python tools/ncu_summary.py gpurun_out/warm_c4.csv 2 > gpurun_out/warm_c4.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_hier.csv python tools/one_hier.py 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_hier.csv 1 > gpurun_out/hier.txt
