"""Cut-link pass counters per bench workload (lines recorded vs capacity,
overflow faces, band candidates).  usage: python tools/link_stats.py c2 c4"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_01251_b200.voxelizer import EmbedEngine  # noqa: E402

for name in sys.argv[1:] or ["c2"]:
    w = bench.WORKLOADS[name]
    eng = EmbedEngine(bench.make_mesh(w, 0), bench.make_cfg(w), use_graph=False)
    eng.run()
    st = eng.link_stats()
    st["faces"] = int(eng.mesh.n_faces)
    st["lines_per_face"] = st["lines"] / st["faces"]
    print(name, json.dumps(st))
