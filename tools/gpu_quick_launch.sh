#!/bin/bash
# warm-cache ncu launch lists of C2 and C4 (one_embed.py), summarised per kernel
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for c in ${@:-c2 c4}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/warm_$c.csv python tools/one_embed.py $c 2 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/warm_$c.csv 2 > gpurun_out/warm_$c.txt
done
