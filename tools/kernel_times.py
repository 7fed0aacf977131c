"""Per-kernel device times of one eager embed (EmbedEngine.kernel_times, all
kernels on one stream) for the bench workloads: JSON per config.
  python tools/kernel_times.py c2 c4"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import torch  # noqa: E402
from paper_2512_01251_b200.voxelizer import EmbedEngine  # noqa: E402

for c in sys.argv[1:] or ["c2"]:
    w = bench.WORKLOADS[c]
    eng = EmbedEngine(bench.make_mesh(w, 0), bench.make_cfg(w))
    for _ in range(3):
        eng.run()
    kt = [eng.kernel_times() for _ in range(3)]
    med = {k: (kt[0][k][0], sorted(x[k][1] for x in kt)[1]) for k in kt[0]}
    tot = sum(v[1] for v in med.values())
    print(json.dumps({"config": c, "total_ms": tot,
                      "kernels": {k: {"launches": v[0], "ms": round(v[1], 4)} for k, v in
                                  sorted(med.items(), key=lambda kv: -kv[1][1])}}), flush=True)
