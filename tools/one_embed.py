"""Run warm-up embeds then one embed (for ncu -k ... -c 1 captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_01251_b200 import EmbedConfig, make_icosphere, make_torus
from paper_2512_01251_b200.voxelizer import EmbedEngine
which = sys.argv[1] if len(sys.argv) > 1 else "c2"
if which == "c1":
    mesh, cfg = make_icosphere((0.5, 0.5, 0.5), 0.5, 5), EmbedConfig(n_x=64, l_max=3)
elif which == "c2":
    mesh, cfg = make_torus(280, 200), EmbedConfig(n_x=64, l_max=4)
else:
    mesh, cfg = make_torus(3000, 1200), EmbedConfig(n_x=64, l_max=5)
eng = EmbedEngine(mesh, cfg)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for _ in range(n):
    eng.run()
torch.cuda.synchronize()
print("done", eng.grid.n_used)
