"""Warm per-kernel device times of the C3 LBM (vf_ktimer over 10 steps per
level and over one eager coarse step of the hierarchy)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_01251_b200 import _lib  # noqa: E402
from paper_2512_01251_b200.solver import FlowConfig, LbmHierarchy, LbmLevel  # noqa: E402
from paper_2512_01251_b200.voxelizer import EmbedEngine  # noqa: E402

w = bench.WORKLOADS["c3"]
eng = EmbedEngine(bench.make_mesh(w, 0), bench.make_cfg(w))
grid, table = eng.run()
lib = _lib.require_cuda()


def timed(fn, label):
    torch.cuda.synchronize()
    _lib.check(lib.vf_ktimer_start(_lib.stream_ptr(), 2000.0), "kt")
    fn()
    buf = C.create_string_buffer(1 << 16)
    lib.vf_ktimer_stop(buf, len(buf))
    print(label)
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split("\t")
        print(f"  {name:24s} n={int(cnt):3d} mean={1e3 * float(ms) / int(cnt):8.2f} us")


Lf = grid.n_levels - 1
for L in range(grid.n_levels):
    lv = LbmLevel(grid, L, table if L == Lf else None,
                  FlowConfig(Re=20.0, u_in=0.05, D_s=8.0, bc_scheme="IBB" if L == Lf else "SBB"))
    lv.init_equilibrium(1.0, (0.05, 0, 0)).step(3, force=False)
    timed(lambda: lv.step(10, force=(L == Lf)), f"level {L}")
h = LbmHierarchy(grid, table, FlowConfig(Re=20.0, u_in=0.05, D_s=8.0, bc_scheme="IBB"), order=3)
h.init_equilibrium(1.0, (0.05, 0, 0)).step(2)
timed(lambda: h.step(1), "hierarchy coarse step (eager)")
