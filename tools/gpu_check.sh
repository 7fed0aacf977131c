#!/bin/bash
# One GPU session: parity tests, smoke, bench (C2 + C4), launch list, ncu --set full of the top kernels.
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python tools/quick_embed.py c1 c2 c4 > gpurun_out/quick.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config c4 --steps 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
if [ -n "$NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/one_embed.py c2 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_links|k_voxelize|k_indicators|k_pairs|k_adapt_children" -s 21 -c 21 -o gpurun_out/prof_c2 -f python tools/one_embed.py c2 2 > gpurun_out/ncu_c2.log 2>&1
fi
ls -la gpurun_out
