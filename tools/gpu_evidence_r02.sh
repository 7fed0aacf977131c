#!/bin/bash
# Round-2 evidence on one B200: bench lines (C4 default, C2, C3, the reference
# arm), ncu launch list of a C4 embed, and an ncu --set full capture of one
# steady-state C4 embed summarised per kernel into profiles/ncu_traffic.json.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err
timeout 600 python bench.py --config c2 > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
timeout 600 python bench.py --config c3 > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c4.csv python tools/one_embed.py c4 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_launches_c4.csv 2 > gpurun_out/r02_launches_c4.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r02_launches_c4_warm.csv python tools/one_embed.py c4 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_launches_c4_warm.csv 2 > gpurun_out/r02_launches_c4_warm.txt
# one steady-state embed: skip the first run's launches (LUT sizing run + eager run)
NL=$(python -c "import csv; r=list(csv.reader(open('gpurun_out/r02_launches_c4.csv'))); h=[i for i,x in enumerate(r) if 'Kernel Name' in x][0]; print(len(r)-h-1)")
SKIP=$((NL - 80))
echo "launches $NL skip $SKIP" > gpurun_out/r02_ncu_full.log
timeout 1500 ncu --set full --clock-control none -s $SKIP -c 80 -o /tmp/full_c4 -f python tools/one_embed.py c4 2 >> gpurun_out/r02_ncu_full.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json 2>/dev/null
python tools/ncu_traffic.py /tmp/full_c4.ncu-rep c4 > gpurun_out/r02_ncu_full_c4.txt 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_new.json
# (reference arm: run separately, ~4 min)
tail -c 400 gpurun_out/r02_bench_c4.json; cat gpurun_out/r02_ncu_full_c4.txt | head -40
