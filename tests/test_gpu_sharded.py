"""Block-sharded multi-GPU embed vs the single-GPU embed.  Only one GPU is
available to the test harness, so two ranks share cuda:0 over a gloo group
(the exchange code path is the same as with NCCL across GPUs).  Topology and
flags must be identical on every rank; masks and LUT slots of the blocks a rank
owns must be bit-identical to the single-GPU result."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_01251_b200 import EmbedConfig, make_torus
        from paper_2512_01251_b200.mesh import translate
        from paper_2512_01251_b200.parallel import ShardedEmbed
        from paper_2512_01251_b200.voxelizer import EmbedEngine
        mesh = translate(make_torus(120, 60), (0.0031, -0.0017, 0.0023))
        cfg = EmbedConfig(n_x=32, l_max=4)
        ref_g, ref_t = EmbedEngine(mesh, cfg, use_graph=False).run()
        R = ref_g.to_numpy()
        ref_len = ref_t.lengths.cpu().numpy()
        ref_cmap = ref_t.contraction_map.cpu().numpy()[:ref_g.n_used]
        sh = ShardedEmbed(mesh, cfg, capacity=ref_g.capacity)
        g, t = sh.run()
        G = g.to_numpy()
        errs = []
        if not np.array_equal(G["level_start"], R["level_start"]):
            errs.append("level_start")
        for k in ("coords", "nbr", "nbr_child", "child"):
            if not np.array_equal(G[k], R[k]):
                errs.append(k)
        # flags: SOLID/SB/SA/MARK/REFINED replicated; BOUNDARY only on owners
        if not np.array_equal(G["bflags"] & 31, R["bflags"] & 31):
            errs.append("bflags")
        owned_cells = 0
        for L in range(g.n_levels):
            s, e = g.level_range(L)
            own = sh.owned_blocks(L).cpu().numpy()
            if L < g.n_levels - 1:
                # the interface layer of refined blocks is written on owners
                ok = np.array_equal(G["masks"][s:e][own], R["masks"][s:e][own])
            else:
                ok = np.array_equal(G["masks"][s:e][own], R["masks"][s:e][own])
                fl = (G["bflags"][s:e][own] & 32) == (R["bflags"][s:e][own] & 32)
                ok = ok and bool(fl.all())
            if not ok:
                errs.append(f"masks L{L}")
            owned_cells += int(own.sum())
        # the owner map of every level is the balanced contiguous split of the
        # replicated topology (numpy restatement in parallel.balanced_row_owner)
        from paper_2512_01251_b200.parallel import balanced_row_owner
        om = sh.row_owner.cpu().numpy()
        base = 0
        for L in range(g.n_levels):
            s, e = g.level_range(L)
            by, bz = cfg.bins(L)[1], cfg.bins(L)[2]
            co = R["coords"][s:e]
            cnt = np.bincount(co[:, 1] + by * co[:, 2], minlength=by * bz)
            if not np.array_equal(om[base:base + by * bz], balanced_row_owner(cnt, world)):
                errs.append(f"owner map L{L}")
            base += by * bz
        if t.n_b != ref_t.n_b or not np.array_equal(t.contraction_map.cpu().numpy(), ref_cmap):
            errs.append("contraction map")
        Lf = g.n_levels - 1
        s, e = g.level_range(Lf)
        own = sh.owned_blocks(Lf).cpu().numpy()
        slots = ref_cmap[s:e][own]
        slots = slots[slots >= 0]
        lg = t.lengths.cpu().numpy()
        if not np.array_equal(lg[slots], ref_len[slots]):
            errs.append("lengths")
        q.put((rank, errs, owned_cells, len(slots), sh.comm_bytes))
    except Exception as ex:  # report instead of hanging the parent
        q.put((rank, [repr(ex)], 0, 0, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_embed_matches_single_gpu(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for r in res:
        assert r[1] == [], r
    assert all(r[3] > 0 for r in res)  # every rank owns LUT slots


def test_native_nccl_single_rank():
    """The native driver (vf_shard_embed_phase1: the exchanges on the
    library's NCCL communicator, no host sync) on a 1-rank communicator --
    the only NCCL world one GPU allows -- equals the single-GPU embed
    bitwise, eager and replayed from a CUDA graph of phase 1."""
    from paper_2512_01251_b200 import EmbedConfig, make_torus
    from paper_2512_01251_b200.mesh import translate
    from paper_2512_01251_b200.parallel import NcclShardedEmbed, nccl_unique_id
    from paper_2512_01251_b200.voxelizer import EmbedEngine
    mesh = translate(make_torus(120, 60), (0.0031, -0.0017, 0.0023))
    cfg = EmbedConfig(n_x=32, l_max=4)
    ref_g, ref_t = EmbedEngine(mesh, cfg, use_graph=False).run()
    R = ref_g.to_numpy()
    sh = NcclShardedEmbed(mesh, cfg, 0, 1, nccl_unique_id(), capacity=ref_g.capacity)
    g, t = sh.run()

    def check(g, t):
        G = g.to_numpy()
        assert np.array_equal(G["level_start"], R["level_start"])
        for k in ("coords", "nbr", "nbr_child", "child", "bflags", "masks"):
            assert np.array_equal(G[k][:ref_g.n_used], R[k][:ref_g.n_used]), k
        assert t.n_b == ref_t.n_b
        assert np.array_equal(t.contraction_map.cpu().numpy(), ref_t.contraction_map.cpu().numpy()[:ref_g.n_used])
        assert np.array_equal(t.lengths.cpu().numpy(), ref_t.lengths.cpu().numpy())

    check(g, t)
    # phase 1 captured into a CUDA graph (kernels + NCCL all-reduces) and replayed
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        sh.phase1()  # warm-up on the capture stream
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            sh.phase1(stream=s)
    torch.cuda.current_stream().wait_stream(s)
    sh.grid.masks.zero_()
    sh.grid.bflags.zero_()
    sh.cmap.fill_(-7)
    graph.replay()
    torch.cuda.synchronize()
    G = sh.grid.to_numpy()
    for k in ("coords", "nbr", "nbr_child", "child", "bflags", "masks"):
        assert np.array_equal(G[k][:ref_g.n_used], R[k][:ref_g.n_used]), k
    assert int(sh.nb_dev.item()) == ref_t.n_b
    assert np.array_equal(sh.cmap.cpu().numpy()[:ref_g.n_used], ref_t.contraction_map.cpu().numpy()[:ref_g.n_used])
