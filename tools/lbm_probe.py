"""C3 LBM probe: embed the C3 sphere, then bench.lbm_block (per-level
collide/stream times + one hierarchy coarse step).  Also the ncu driver for
the LBM kernels:  tools/lbm_probe.py [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_01251_b200.voxelizer import EmbedEngine  # noqa: E402

w = bench.WORKLOADS["c3"]
eng = EmbedEngine(bench.make_mesh(w, 0), bench.make_cfg(w))


class A:
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10


flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
r = bench.lbm_block(eng, w, A, flush)
print(json.dumps({"levels": [(d["level"], round(d["step_ms"], 4), round(d["hbm_frac"], 3)) for d in r["levels"]],
                  "coarse_step_ms": r["coarse_step_ms"], "levels_only": r["coarse_step_ms_levels_only"],
                  "force": r["wall_force_lattice"]}))
# blocks with a non-simple cell per level (k_lbm_special's list)
from paper_2512_01251_b200.solver import FlowConfig, LbmLevel  # noqa: E402
grid, table = eng.run()
for L in range(grid.n_levels):
    lv = LbmLevel(grid, L, table if L == grid.n_levels - 1 else None, FlowConfig(Re=20.0, u_in=0.05, D_s=8.0))
    lv.init_equilibrium(1.0, (0.05, 0, 0)).step(1, force=False)
    s, e = grid.level_range(L)
    print(f"level {L}: blocks {e - s}, special {int(lv.scratch[0].item())}")
