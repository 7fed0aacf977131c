#!/bin/bash
# iteration run: GPU parity tests (optionally -k filtered) + stage timings + bench (optional)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout ${PYT_TIMEOUT:-1200} python -m pytest tests -q -m gpu -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_embed.py c1 c2 c4 > gpurun_out/quick.log 2>&1; cat gpurun_out/quick.log | tail -8
if [ -n "$BENCH" ]; then timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step']); print(d['config']['stage_ms_serial']); [print(k['kernel'], round(k['ms_per_embed'],4), round(k['frac'],3)) for k in d['roofline']['kernels']]"; fi
if [ -n "$LAUNCH" ]; then timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/one_embed.py c4 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_c4.csv 2 > gpurun_out/launches_c4.txt; head -30 gpurun_out/launches_c4.txt; fi
