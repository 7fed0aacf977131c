"""Scratch timing of the embed pipeline (not the bench contract)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_01251_b200 import EmbedConfig, make_icosphere, make_torus
from paper_2512_01251_b200.voxelizer import EmbedEngine

def run(name, mesh, cfg, reps=10):
    eng = EmbedEngine(mesh, cfg)
    for _ in range(3):
        eng.run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        eng.run(timed=True)
        torch.cuda.synchronize()
        ts.append(eng.timings())
    t = sorted(ts, key=lambda x: x.total)[len(ts) // 2]
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gt = []
    for _ in range(reps):
        s.record(); eng.run(); e.record(); torch.cuda.synchronize(); gt.append(s.elapsed_time(e))
    gt.sort()
    print(f"{name}: F={mesh.n_faces} blocks={eng.grid.n_used} n_b={int(eng.n_b_host[0])} "
          f"eager={t.total:.3f}ms bins={t.binning:.3f} vox={t.voxelization:.3f} "
          f"ref={t.refinement:.3f} bnd={t.boundary:.3f} links={t.links:.3f} (k_links {eng.link_kernel_ms():.3f}) "
          f"| graph={gt[len(gt)//2]:.3f}ms", flush=True)

if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2"]
    if "c1" in which:
        run("C1", make_icosphere((0.5,0.5,0.5),0.5,5), EmbedConfig(n_x=64, l_max=3))
    if "c2" in which:
        run("C2", make_torus(280, 200), EmbedConfig(n_x=64, l_max=4))
    if "c4" in which:
        run("C4", make_torus(3000, 1200), EmbedConfig(n_x=64, l_max=5), reps=5)
