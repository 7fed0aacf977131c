"""C5 sweep: torus meshes 10K..7.2M faces x L_max 3..6 on one
GPU -- embed time (steady state, L2 flushed between runs, CUDA events),
cells classified/s, blocks, boundary blocks, post-refine_faces F.

  python tools/sweep_c5.py [--lmax 3,4,5,6] [--meshes 100x50,...] > c5.jsonl"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2512_01251_b200 import EmbedConfig, make_torus, l_spec_bound, refine_faces  # noqa: E402
from paper_2512_01251_b200.voxelizer import EmbedEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lmax", default="3,4,5,6")
ap.add_argument("--meshes", default="100x50,280x200,700x500,1500x800,3000x1200")
ap.add_argument("--runs", type=int, default=5)
a = ap.parse_args()
flush = torch.empty(64 << 20, device="cuda")
for ms in a.meshes.split(","):
    m, n = map(int, ms.split("x"))
    base = make_torus(m, n)
    for L in map(int, a.lmax.split(",")):
        cfg = EmbedConfig(n_x=64, l_max=L, n_spec=2, d_spec=0.05)
        t0 = time.perf_counter()
        mesh = refine_faces(base, l_spec_bound(cfg.domain, cfg.n_spec, L, cfg.nb[0]))
        t_ref = time.perf_counter() - t0
        rec = {"mesh": f"torus {m}x{n}", "faces_in": int(base.n_faces), "faces": int(mesh.n_faces), "l_max": L,
               "refine_faces_s": round(t_ref, 3)}
        try:
            eng = EmbedEngine(mesh, cfg)
            for _ in range(2):
                eng.run()
            torch.cuda.synchronize()
            st = eng.stream
            ts = []
            for k in range(a.runs):
                flush.fill_(float(k))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(st)
                g, tab = eng.run()
                e1.record(st)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            cells = eng.cells_classified()
            ms_ = float(np.median(ts))
            rec.update({"embed_ms": round(ms_, 4), "cells": int(cells), "cells_per_s": cells / (ms_ / 1e3),
                        "blocks": int(g.n_used), "boundary_blocks": int(tab.n_b), "capacity": int(g.capacity),
                        "graph": bool(eng.use_graph)})
            del eng, g, tab
        except Exception as ex:  # capacity / memory: record and go on
            rec["error"] = f"{type(ex).__name__}: {ex}"[:200]
        torch.cuda.empty_cache()
        print(json.dumps(rec), flush=True)
