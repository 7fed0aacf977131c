"""Embed C3 and run a few LBM steps on one level (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_01251_b200 import EmbedConfig, make_icosphere
from paper_2512_01251_b200.solver import FlowConfig, LbmLevel
from paper_2512_01251_b200.voxelizer import EmbedEngine
L = int(sys.argv[1]) if len(sys.argv) > 1 else 0
mesh = make_icosphere((0.5, 0.5, 0.5), 1.0 / 64, 5)
grid, table = EmbedEngine(mesh, EmbedConfig(n_x=128, l_max=3)).run()
Lf = grid.n_levels - 1
lv = LbmLevel(grid, L, table if L == Lf else None,
              FlowConfig(u_in=0.05, D_s=8.0 / 2 ** (Lf - L), bc_scheme="IBB" if L == Lf else "SBB"))
lv.init_equilibrium(1.0, (0.05, 0, 0))
lv.step(5)
torch.cuda.synchronize()
print("ok", lv.s, lv.e)
