"""C5 depth check: the 7.2M-face torus embedded at L_max = 5, 6, 7 on one GPU:
time per embed (eager, median of 3 after a warm-up), blocks, boundary blocks,
embed workspace and peak device memory.  usage: python tools/deep_embed.py [lmax ...]"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2512_01251_b200 import EmbedConfig, make_torus  # noqa: E402
from paper_2512_01251_b200.voxelizer import EmbedEngine  # noqa: E402

mesh = make_torus(3000, 1200)
for lm in [int(a) for a in sys.argv[1:]] or [5, 6, 7]:
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    cfg = EmbedConfig(n_x=64, l_max=lm)
    eng = EmbedEngine(mesh, cfg)
    eng.run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        eng.run()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    n_used = int(eng.grid.level_start[eng.grid.n_levels].item())
    print(json.dumps({"l_max": lm, "faces": mesh.n_faces, "blocks": n_used, "cells": 64 * n_used,
                      "boundary_blocks": int(eng.n_b_host[0]), "embed_ms": sorted(ts)[1],
                      "gcells_per_s": 64 * n_used / sorted(ts)[1] / 1e6,
                      "workspace_gb": eng.ws.numel() / 1e9, "capacity": eng.grid.capacity,
                      "peak_gb": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
    del eng
