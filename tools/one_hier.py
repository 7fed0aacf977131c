"""C3 embed + n eager step_hierarchy coarse steps (for ncu launch lists).
usage: python tools/one_hier.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2512_01251_b200.solver import FlowConfig, LbmHierarchy  # noqa: E402
from paper_2512_01251_b200.voxelizer import EmbedEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = bench.WORKLOADS["c3"]
eng = EmbedEngine(bench.make_mesh(w, 0), bench.make_cfg(w), use_graph=False)
grid, table = eng.run()
Lf = grid.n_levels - 1
D_f = w["diameter"] * 4 * w["n_x"] // 4 * 2 ** Lf
h = LbmHierarchy(grid, table, FlowConfig(Re=20.0, u_in=0.05, D_s=D_f / 2 ** Lf)).init_equilibrium(1.0, (0.05, 0, 0))
h.step(n)
torch.cuda.synchronize()
print("ranges", [grid.level_range(L) for L in range(grid.n_levels)])
