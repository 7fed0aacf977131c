"""Amdahl model of the block-sharded embed from measured
1-GPU kernel times: the native sharded pipeline (vf_shard_embed_phase1 on a
1-rank NCCL communicator, every row owned) runs under the per-kernel timer;
kernels whose work is split by row ownership are 'partitioned', the rest
(replicated topology, per-level face scans, tables) 'replicated'.  Projected
T(N) = T_rep + T_part / N + T_comm(N), with T_comm from the all-reduce sizes
over an NVLink/NVSwitch ring bus bandwidth plus a per-call latency.
usage: python tools/shard_model.py [c4]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2512_01251_b200 import _lib  # noqa: E402
from paper_2512_01251_b200.parallel import NcclShardedEmbed, nccl_unique_id  # noqa: E402

# split by row ownership: owned bins / blocks / rows, the faces near owned
# rows (cut links), the owned LUT slots
PART = {"k_pairs", "k_pair_blocks", "k_pair_scatter", "k_voxelize", "k_xrows", "k_boundary",
        "k_links_small", "k_links_enum", "k_links_q", "k_block_count", "k_block_scatter", "k_lut_blocks",
        "k_links_band", "k_links_ovf", "k_links_full", "k_face_near_owned"}
w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
mesh, cfg = bench.make_mesh(w, 0), bench.make_cfg(w)
sh = NcclShardedEmbed(mesh, cfg, 0, 1, nccl_unique_id())
for _ in range(2):
    sh.run()
torch.cuda.synchronize()
lib = sh.lib
st = _lib.stream_ptr()
_lib.check(lib.vf_ktimer_start(st, 3000.0), "ktimer")
try:
    gs = sh.phase1()
    _lib.check(lib.vf_shard_links(C.byref(sh.c), _lib.ptr(sh.mesh.faces), sh.mesh.n_faces, C.byref(gs),
                                  _lib.ptr(sh.cmap), _lib.ptr(sh.nb_dev), _lib.ptr(sh.lengths),
                                  sh.lengths.shape[0], _lib.ptr(sh.ws), sh.ws.numel(), st), "links")
finally:
    buf = C.create_string_buffer(1 << 16)
    n = lib.vf_ktimer_stop(buf, len(buf))
kt = {}
for line in buf.value.decode().splitlines():
    name, cnt, ms = line.split("\t")
    kt[name] = (int(cnt), float(ms))
part = sum(v[1] for k, v in kt.items() if k in PART)
rep = sum(v[1] for k, v in kt.items() if k not in PART)
cap = sh.grid.capacity
# all-reduce bytes per embed: L_max x 1 B flags + 8 B SOLID masks + 4 B counts per block of capacity
ar_bytes = cap * (cfg.l_max + 12)
n_calls = cfg.l_max + 2
out = {"workload": w["desc"], "t_replicated_ms": rep, "t_partitioned_ms": part,
       "allreduce_bytes": ar_bytes, "allreduce_calls": n_calls,
       "kernels": {k: round(v[1], 4) for k, v in sorted(kt.items(), key=lambda kv: -kv[1][1])}}
proj = {}
for N in (1, 2, 4, 8):
    # ring all-reduce moves 2 (N-1)/N of the buffer over each GPU's NVLink
    # (~450 GB/s effective per direction measured class); ~15 us per call
    comm = 0.0 if N == 1 else (2 * (N - 1) / N * ar_bytes / 450e9 * 1e3 + n_calls * 0.015)
    t = rep + part / N + comm
    proj[N] = {"ms": round(t, 4), "comm_ms": round(comm, 4), "speedup": round((rep + part) / t, 3)}
out["projection"] = proj
print(json.dumps(out))
