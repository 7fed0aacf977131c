#!/bin/bash
# Quick GPU iteration: parity tests (-m gpu), stage timings, optional bench / ncu.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_embed.py c1 c2 c4 2>&1 | tee gpurun_out/quick.log
if [ -n "$BENCH" ]; then timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json; fi
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s ${NCU_S:-0} -c ${NCU_C:-1} -o gpurun_out/prof -f python tools/one_embed.py ${NCU_CFG:-c2} 2 > gpurun_out/ncu.log 2>&1; tail -2 gpurun_out/ncu.log
fi
