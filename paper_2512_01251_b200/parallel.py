"""parallel -- block-sharded multi-GPU embed (BASELINE north star: grid blocks
partitioned across the GPUs of one box, mesh replicated on every GPU, NCCL over
NVLink used only for per-level flags and counts).

One process per GPU (torchrun), ``torch.distributed`` process group (NCCL; gloo
works too, which is how the CPU/1-GPU tests exercise it).

Ownership: whole level-L block rows (j, k) -- hence every x-run of Alg. 5 --
belong to one rank.  The rows are cut into contiguous ranges (row = j + B_y k)
holding equal numbers of level-L blocks (``vf_shard_owner_map``, computed from
the replicated topology, so every rank derives the same map without
communication).  A face then touches the rows of one or two ranks.  Per level
every rank
  1. bins only faces that hit one of ITS rows and only ITS bins, voxelizes,
     and runs Alg. 5 (+x, -x) + finalize on its rows (``vf_shard_level``,
     exact because runs never leave a row);
  2. zeroes the level's block flags of rows it does not own and all-reduces
     them (MAX over uint8, 1 B/block): every rank now holds the exact solid
     flags of the whole level;
  3. marks and adapts REPLICATED (deterministic, identical on every rank) and
     derives the next level's owner map (``vf_shard_refine``), so the block
     topology is identical everywhere without any exchange.
At the finest level the exchange adds the 64-bit SOLID-cell masks (SUM over
owner-zeroed int64, 8 B/block) for the boundary halo and, after boundary
detection on owned blocks, the per-block boundary counts (SUM, 4 B/block)
for the global contraction map.  Link lengths are computed for owned blocks
only, from the faces near owned rows (~F/N per rank): the LUT stays
distributed (rank r holds the slots of its blocks), as a sharded solver
consumes it.

Results on owned data are bit-identical to the single-GPU embed
(tests/test_gpu_sharded.py); topology and flags are identical on every rank.

Two drivers run this schedule:
  * ``NcclShardedEmbed`` -- the NATIVE one: ``vf_shard_embed_phase1`` runs every
    level and issues the exchanges itself on the library's NCCL communicator
    (MAX all-reduces over owner-zeroed arrays, stream-ordered, no host sync,
    graph-capturable); used when the process group's backend is NCCL;
  * ``ShardedEmbed`` over any torch.distributed backend (the stage calls with
    ``dist.all_reduce`` between them); on an NCCL group it delegates to the
    native driver, on gloo (CPU tests, several ranks sharing one GPU) it runs
    the exchanges from Python.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .config import EmbedConfig
from .datatypes import ForestGrid, LinkTable, as_device_mesh


def row_owner(j, k, by_L: int, n_ranks: int):
    """Owner rank of level-L block row(s) (j, k); by_L = blocks per axis y."""
    if n_ranks <= 1:
        return np.zeros_like(np.asarray(j))
    return (np.asarray(j, dtype=np.int64) + by_L * np.asarray(k, dtype=np.int64)) % n_ranks


def balanced_row_owner(counts, n_ranks: int):
    """numpy restatement of vf_shard_owner_map (k_row_assign): owner of each
    block row = the rank whose 1/N share of the level's blocks holds the row's
    first block.  ``counts`` = blocks per row (row = j + B_y k)."""
    counts = np.asarray(counts, dtype=np.int64)
    total = int(counts.sum())
    if n_ranks <= 1 or total == 0:
        return np.zeros(counts.shape, dtype=np.uint8)
    excl = np.cumsum(counts) - counts
    return np.minimum(excl * n_ranks // total, n_ranks - 1).astype(np.uint8)


def owner_zero_allreduce(t, owned_mask, op, group=None):
    """Publish owner values: zero what this rank does not own, then one
    all-reduce (MAX for non-negative flags, SUM for bit masks / counts)."""
    import torch.distributed as dist
    t.masked_fill_(~owned_mask, 0)
    dist.all_reduce(t, op=op, group=group)
    return t


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it, the ranks share it)."""
    lib = _lib.require_cuda()
    buf = (C.c_char * 128)()
    _lib.check(lib.vf_nccl_unique_id(buf, 128), "vf_nccl_unique_id")
    return bytes(buf)


class NcclShardedEmbed:
    """Native block-sharded embed of one rank: the library's NCCL
    communicator (``vf_ctx_create_nccl``) carries the per-level exchanges
    inside ``vf_shard_embed_phase1`` (no host synchronisation until the LUT
    is sized), then ``vf_shard_links`` fills the LUT slots of owned blocks."""

    def __init__(self, mesh, cfg: EmbedConfig, rank: int, world: int, unique_id: bytes,
                 capacity: Optional[int] = None):
        import torch
        self.torch = torch
        self.lib = _lib.require_cuda()
        self.rank, self.world = int(rank), int(world)
        self.cfg = cfg
        self.mesh = as_device_mesh(mesh)
        cap = int(capacity if capacity is not None else cfg.block_capacity(self.mesh.area))
        self.grid = ForestGrid.allocate(cfg, cap)
        self.c = _lib.make_config(cfg, shard=(self.rank, self.world))
        nown = self.lib.vf_shard_owner_bytes(C.byref(self.c))
        self.row_owner = torch.zeros(max(int(nown), 1), dtype=torch.uint8, device="cuda")
        self.c.d_row_owner = self.row_owner.data_ptr()
        wsb = self.lib.vf_embed_workspace_size(C.byref(self.c), self.mesh.n_faces, cap)
        if wsb == 0:
            raise ValueError("invalid embed configuration")
        self.ws = torch.empty(int(wsb), dtype=torch.uint8, device="cuda")
        self.bcount = torch.empty(cap, dtype=torch.int32, device="cuda")
        self.cmap = torch.empty(cap, dtype=torch.int32, device="cuda")
        self.nb_dev = torch.zeros(1, dtype=torch.int32, device="cuda")
        uid = (C.c_char * 128).from_buffer_copy(unique_id)
        self.ctx = self.lib.vf_ctx_create_nccl(torch.cuda.current_device(), self.world, self.rank, uid)
        if not self.ctx:
            raise _lib.CudaError(f"vf_ctx_create_nccl: {_lib.last_error()}")
        self.lengths = None
        self.bc_ids = None
        # bytes all-reduced per embed: L_max x capacity flags + 8 B SOLID
        # masks + 4 B boundary counts per block of capacity
        self.comm_bytes = cap * (cfg.l_max + 8 + 4)

    def __del__(self):
        try:
            if self.ctx:
                self.lib.vf_ctx_destroy(self.ctx)
        except Exception:
            pass

    def phase1(self, use_filter: Optional[bool] = None, stream=None):
        """Every level + exchanges + tables, enqueued on ``stream`` (no sync)."""
        g, c = self.grid, self.c
        uf = int(bool(self.cfg.use_filter if use_filter is None else use_filter))
        g.status.zero_()
        gs = g._struct()
        _lib.check(self.lib.vf_shard_embed_phase1(
            self.ctx, C.byref(c), _lib.ptr(self.mesh.faces), self.mesh.n_faces, uf, C.byref(gs),
            _lib.ptr(self.bcount), _lib.ptr(self.cmap), _lib.ptr(self.nb_dev), _lib.ptr(self.ws),
            self.ws.numel(), _lib.stream_ptr(stream)), "embed_geometry (native sharded)")
        g.n_levels = self.cfg.l_max
        return gs

    def run(self, use_filter: Optional[bool] = None):
        torch, lib, g, c = self.torch, self.lib, self.grid, self.c
        gs = self.phase1(use_filter)
        st = _lib.stream_ptr()
        _lib.check(lib.vf_check_status(C.byref(gs), st), "embed_geometry (native sharded)")
        n_b = int(self.nb_dev.item())
        if self.lengths is None or self.lengths.shape[0] < n_b:
            cap = int(n_b * 1.25) + 16
            self.lengths = torch.empty((cap, 27, 64), dtype=torch.float32, device="cuda")
            self.bc_ids = torch.zeros((cap, 27, 64), dtype=torch.int8, device="cuda")
        _lib.check(lib.vf_shard_links(C.byref(c), _lib.ptr(self.mesh.faces), self.mesh.n_faces, C.byref(gs),
                                      _lib.ptr(self.cmap), _lib.ptr(self.nb_dev), _lib.ptr(self.lengths),
                                      self.lengths.shape[0], _lib.ptr(self.ws), self.ws.numel(), st),
                   "link lengths")
        _lib.check(lib.vf_check_status(C.byref(gs), st), "embed_geometry (native sharded links)")
        return g, LinkTable(self.lengths[:n_b], self.bc_ids[:n_b], self.cmap[:g.n_used], n_b)

    def owned_blocks(self, L: int):
        s, e = self.grid.level_range(L)
        co = self.grid.coords[s:e].long()
        by = self.cfg.bins(L)[1]
        base = sum(self.cfg.bins(l)[1] * self.cfg.bins(l)[2] for l in range(L))
        return self.row_owner[base + co[:, 1] + by * co[:, 2]] == self.rank

    def cells_classified(self) -> int:
        return 64 * self.grid.n_used


class ShardedEmbed:
    """embed_geometry split across the ranks of a process group (NCCL group:
    the native driver; other backends: Python-driven exchanges)."""

    def __new__(cls, mesh, cfg: EmbedConfig, group=None, capacity: Optional[int] = None,
                native: Optional[bool] = None):
        import torch.distributed as dist
        if native is None:
            native = dist.get_backend(group) == "nccl"
        if not native:
            return super().__new__(cls)
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return NcclShardedEmbed(mesh, cfg, rank, world, obj[0], capacity)

    def __init__(self, mesh, cfg: EmbedConfig, group=None, capacity: Optional[int] = None,
                 native: Optional[bool] = None):
        import torch
        import torch.distributed as dist
        self.torch = torch
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.lib = _lib.require_cuda()
        self.cfg = cfg
        self.mesh = as_device_mesh(mesh)
        cap = int(capacity if capacity is not None else cfg.block_capacity(self.mesh.area))
        self.grid = ForestGrid.allocate(cfg, cap)
        self.c = _lib.make_config(cfg, shard=(self.rank, self.world))
        nown = self.lib.vf_shard_owner_bytes(C.byref(self.c))
        self.row_owner = torch.zeros(max(int(nown), 1), dtype=torch.uint8, device="cuda")
        self.c.d_row_owner = self.row_owner.data_ptr()
        F = self.mesh.n_faces
        wsb = self.lib.vf_embed_workspace_size(C.byref(self.c), F, cap)
        if wsb == 0:
            raise ValueError("invalid embed configuration")
        self.ws = torch.empty(int(wsb), dtype=torch.uint8, device="cuda")
        self.bcount = torch.empty(cap, dtype=torch.int32, device="cuda")
        self.cmap = torch.empty(cap, dtype=torch.int32, device="cuda")
        self.scal = torch.zeros(8, dtype=torch.int32, device="cuda")
        self.tab_ws = torch.empty(int(self.lib.vf_tables_workspace_size(C.byref(self.grid._struct()))),
                                  dtype=torch.uint8, device="cuda")
        self.lengths = None
        self.bc_ids = None
        self.comm_bytes = 0

    def _owned(self, L, s, e):
        co = self.grid.coords[s:e].long()
        by = self.cfg.bins(L)[1]
        rows = co[:, 1] + by * co[:, 2]
        base = sum(self.cfg.bins(l)[1] * self.cfg.bins(l)[2] for l in range(L))
        return self.row_owner[base + rows] == self.rank

    # -- the sharded pipeline ----------------------------------------------
    def run(self, use_filter: Optional[bool] = None):
        torch, dist, lib = self.torch, self.dist, self.lib
        cfg, g, c = self.cfg, self.grid, self.c
        uf = int(bool(cfg.use_filter if use_filter is None else use_filter))
        st = _lib.stream_ptr()
        faces, F = _lib.ptr(self.mesh.faces), self.mesh.n_faces
        ws, wsn = _lib.ptr(self.ws), self.ws.numel()
        g.status.zero_()
        gs = g._struct()
        _lib.check(lib.vf_init_forest(C.byref(c), C.byref(gs), st), "init_forest")
        g.n_levels = gs.n_levels
        _lib.check(lib.vf_shard_owner_map(C.byref(c), C.byref(gs), 0, ws, wsn, st), "owner map")
        self.comm_bytes = 0
        for L in range(cfg.l_max):
            gs = g._struct()
            _lib.check(lib.vf_shard_level(C.byref(c), faces, F, uf, C.byref(gs), L, ws, wsn, st),
                       "shard level")
            s, e = g.level_range(L)
            # exchange: level flags (1 B/block); finest level also SOLID masks
            dist.all_reduce(g.bflags[s:e], op=dist.ReduceOp.MAX, group=self.group)
            self.comm_bytes += (e - s)
            if L == cfg.l_max - 1:
                dist.all_reduce(g.solid64[s:e], op=dist.ReduceOp.SUM, group=self.group)
                self.comm_bytes += 8 * (e - s)
                break
            _lib.check(lib.vf_shard_refine(C.byref(c), C.byref(gs), L, ws, wsn, st), "shard refine")
            g.n_levels = gs.n_levels
        gs = g._struct()
        Lf = g.n_levels - 1
        s, e = g.level_range(Lf)
        _lib.check(lib.vf_shard_boundary(C.byref(c), C.byref(gs), _lib.ptr(self.bcount), st),
                   "boundary")
        dist.all_reduce(self.bcount[s:e], op=dist.ReduceOp.SUM, group=self.group)
        self.comm_bytes += 4 * (e - s)
        nb_dev = self.scal[4:5]
        _lib.check(lib.vf_link_tables(C.byref(c), C.byref(gs), _lib.ptr(self.bcount),
                                      _lib.ptr(self.cmap), _lib.ptr(nb_dev), _lib.ptr(self.tab_ws),
                                      self.tab_ws.numel(), st), "tables")
        _lib.check(lib.vf_check_status(C.byref(gs), st), "embed_geometry (sharded)")
        n_b = int(nb_dev.item())
        if self.lengths is None or self.lengths.shape[0] < n_b:
            cap = int(n_b * 1.25) + 16
            self.lengths = torch.empty((cap, 27, 64), dtype=torch.float32, device="cuda")
            self.bc_ids = torch.zeros((cap, 27, 64), dtype=torch.int8, device="cuda")
        _lib.check(lib.vf_shard_links(C.byref(c), faces, F, C.byref(gs), _lib.ptr(self.cmap),
                                      _lib.ptr(nb_dev), _lib.ptr(self.lengths), self.lengths.shape[0],
                                      ws, wsn, st), "link lengths")
        _lib.check(lib.vf_check_status(C.byref(gs), st), "embed_geometry (sharded links)")
        return g, LinkTable(self.lengths[:n_b], self.bc_ids[:n_b], self.cmap[:g.n_used], n_b)

    def owned_blocks(self, L: int):
        """Boolean (n_L,) ownership of the level-L blocks (ids in level order)."""
        s, e = self.grid.level_range(L)
        return self._owned(L, s, e)

    def cells_classified(self) -> int:
        return 64 * self.grid.n_used
