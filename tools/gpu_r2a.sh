cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_embed.py c1 c2 c4 > gpurun_out/quick.log 2>&1; cat gpurun_out/quick.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/one_embed.py c4 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_c4.csv 2 > gpurun_out/launches_c4.txt; head -40 gpurun_out/launches_c4.txt
