"""Cut-link kernel time (enumeration + resolution, run alone) vs the
thread-per-face size threshold.  usage: python tools/sweep_small.py c2 c4"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2512_01251_b200 import _lib  # noqa: E402
from paper_2512_01251_b200.voxelizer import EmbedEngine  # noqa: E402

lib = _lib.require_cuda()
lib.vf_set_serial_links(1)
flush = torch.empty(64 << 20, device="cuda")
exts = [float(x) for x in os.environ.get("EXTS", "-1,0.75,1,1.5,2,3,4,6").split(",")]
for name in sys.argv[1:] or ["c2"]:
    w = bench.WORKLOADS[name]
    eng = EmbedEngine(bench.make_mesh(w, 0), bench.make_cfg(w), use_graph=False)
    for e in exts:
        lib.vf_set_link_small_ext(e)
        ms, en = [], []
        for k in range(6):
            flush.fill_(float(k))
            eng.run(timed=True)
            torch.cuda.synchronize()
            if k >= 1:
                ms.append(eng.link_kernel_ms())
                en.append(eng.link_enum_ms())
        st = eng.link_stats()
        print(f"{name} ext={e:5.2f} links {np.median(ms):.4f} ms enum {np.median(en):.4f} ms large {st['large_faces']}",
              flush=True)
