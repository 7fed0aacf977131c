"""Per-step device time of the C4 embed: synchronous run() (one host sync per
embed) vs run_async() (embeds enqueued back to back, validated after)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_01251_b200.voxelizer import EmbedEngine  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
eng = EmbedEngine(bench.make_mesh(w, 0), bench.make_cfg(w))
for _ in range(3):
    eng.run()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
cur = torch.cuda.current_stream()
K = 20
for rep in range(3):
    for mode in ("sync", "async"):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for k in range(K):
            flush.fill_(float(k))
            if mode == "sync":
                eng.run()
            else:
                eng.run_async()
                cur.wait_stream(eng.stream)
        e.record()
        torch.cuda.synchronize()
        if mode == "async":
            eng.check_async()
        print(mode, round(s.elapsed_time(e) / K, 4), "ms per step incl. the L2 flush", flush=True)
