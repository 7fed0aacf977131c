"""parallel -- block-sharded multi-GPU embed (BASELINE north star: grid blocks
partitioned across the GPUs of one box, mesh replicated on every GPU, NCCL over
NVLink used only for per-level flags and counts).

One process per GPU (torchrun), ``torch.distributed`` process group (NCCL; gloo
works too, which is how the CPU/1-GPU tests exercise it).

Ownership: at level L the block row (j, k) -- all blocks with the same (j, k),
hence every x-run of Alg. 5 -- belongs to rank ``(j + B_L,y * k) mod N``
(interleaved for balance; ``row_owner`` mirrors csrc/vf_common.cuh).  Per level
every rank
  1. bins only faces that hit one of ITS rows and only ITS bins
     (vf_build_bins with shard = (rank, N));
  2. voxelizes, propagates (+x, -x) and finalizes -- exact on its rows because
     runs never leave a row;
  3. zeroes the level's block flags of rows it does not own and all-reduces
     them (MAX over uint8, 1 B/block): every rank now holds the exact solid
     flags of the whole level;
  4. marks and adapts REPLICATED (deterministic, identical on every rank), so
     the block topology is identical everywhere without any exchange.
At the finest level the exchange adds the 64-bit SOLID-cell masks (SUM over
owner-zeroed int64, 8 B/block) for the boundary halo and, after boundary
detection on owned blocks, the per-block boundary counts (SUM, 4 B/block)
for the global contraction map.  Link lengths are computed for owned blocks
only: the LUT stays distributed (rank r holds the slots of its blocks), as a
sharded solver consumes it.

Results on owned data are bit-identical to the single-GPU embed
(tests/test_gpu_sharded.py); topology and flags are identical on every rank.
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


def owner_zero_allreduce(t, owned_mask, op, group=None):
    """Publish owner values: zero what this rank does not own, then one
    all-reduce (MAX for non-negative flags, SUM for bit masks / counts)."""
    import torch.distributed as dist
    t.masked_fill_(~owned_mask, 0)
    dist.all_reduce(t, op=op, group=group)
    return t


class ShardedEmbed:
    """embed_geometry split across the ranks of a process group."""

    def __init__(self, mesh, cfg: EmbedConfig, group=None, capacity: Optional[int] = None):
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
        F, Lf = self.mesh.n_faces, cfg.l_max - 1
        nb = cfg.n_bins(Lf)
        dev = "cuda"
        # bins buffers sized for the finest level, reused by every level
        self.counts = torch.empty(nb, dtype=torch.int32, device=dev)
        self.offsets = torch.empty(nb, dtype=torch.int32, device=dev)
        self.face_ids = torch.empty(F * cfg.n_lim, dtype=torch.int32, device=dev)
        self.fmap = torch.empty(F, dtype=torch.int32, device=dev)
        self.scal = torch.zeros(8, dtype=torch.int32, device=dev)
        self.bcount = torch.empty(cap, dtype=torch.int32, device=dev)
        self.cmap = torch.empty(cap, dtype=torch.int32, device=dev)
        gs = self.grid._struct()
        sizes = {
            "bins": max(self.lib.vf_bins_workspace_size(C.byref(self.c), F, L) for L in range(cfg.l_max)),
            "prop": self.lib.vf_propagate_workspace_size(C.byref(gs)),
            "mark": self.lib.vf_mark_workspace_size(C.byref(gs)),
            "adapt": self.lib.vf_adapt_workspace_size(C.byref(gs)),
            "tables": self.lib.vf_tables_workspace_size(C.byref(gs)),
        }
        self.ws = {k: torch.empty(int(v), dtype=torch.uint8, device=dev) for k, v in sizes.items()}
        self.lengths = None
        self.bc_ids = None
        self.comm_bytes = 0

    # -- helpers --------------------------------------------------------
    def _bins_struct(self):
        b = _lib.VfBins()
        b.d_counts, b.d_offsets = self.counts.data_ptr(), self.offsets.data_ptr()
        b.d_face_ids, b.face_ids_cap = self.face_ids.data_ptr(), self.face_ids.numel()
        b.d_n_face_ids = self.scal.data_ptr()
        b.d_map, b.d_n_map = self.fmap.data_ptr(), self.scal.data_ptr() + 4
        return b

    def _owned(self, L, s, e):
        torch = self.torch
        co = self.grid.coords[s:e]
        by = self.cfg.bins(L)[1]
        own = ((co[:, 1].long() + by * co[:, 2].long()) % self.world) == self.rank
        return own

    def _ws(self, k):
        w = self.ws[k]
        return _lib.ptr(w), w.numel()

    # -- the sharded pipeline ----------------------------------------------
    def run(self, use_filter: Optional[bool] = None):
        torch, dist, lib = self.torch, self.dist, self.lib
        cfg, g, c = self.cfg, self.grid, self.c
        uf = int(bool(cfg.use_filter if use_filter is None else use_filter))
        st = _lib.stream_ptr()
        faces, F = _lib.ptr(self.mesh.faces), self.mesh.n_faces
        g.status.zero_()
        gs = g._struct()
        _lib.check(lib.vf_init_forest(C.byref(c), C.byref(gs), st), "init_forest")
        g.n_levels = gs.n_levels
        self.comm_bytes = 0
        b = self._bins_struct()
        status1 = C.c_void_p(self.scal.data_ptr() + 8)
        for L in range(cfg.l_max):
            gs = g._struct()
            _lib.check(lib.vf_build_bins(C.byref(c), faces, F, L, 0, uf, C.byref(b), status1,
                                         *self._ws("bins"), st), "build_bins")
            _lib.check(lib.vf_voxelize_level(C.byref(c), C.byref(gs), L, C.byref(b), faces, st),
                       "voxelize")
            _lib.check(lib.vf_propagate_x(C.byref(c), C.byref(gs), L, +1, int(L == 0),
                                          *self._ws("prop"), st), "propagate +x")
            if L > 0:
                _lib.check(lib.vf_propagate_x(C.byref(c), C.byref(gs), L, -1, 1,
                                              *self._ws("prop"), st), "propagate -x")
            s, e = g.level_range(L)
            # exchange: level flags (1 B/block); finest level also SOLID masks
            _lib.check(lib.vf_shard_zero_unowned(C.byref(c), C.byref(gs), L, None, st), "shard")
            dist.all_reduce(g.bflags[s:e], op=dist.ReduceOp.MAX, group=self.group)
            self.comm_bytes += (e - s)
            if L == cfg.l_max - 1:
                dist.all_reduce(g.solid64[s:e], op=dist.ReduceOp.SUM, group=self.group)
                self.comm_bytes += 8 * (e - s)
                break
            _lib.check(lib.vf_mark_level(C.byref(c), C.byref(gs), L, *self._ws("mark"), st), "mark")
            _lib.check(lib.vf_adapt_refine(C.byref(c), C.byref(gs), L, *self._ws("adapt"), st),
                       "adapt")
            g.n_levels = gs.n_levels
        gs = g._struct()
        Lf = g.n_levels - 1
        s, e = g.level_range(Lf)
        _lib.check(lib.vf_boundary_cells(C.byref(c), C.byref(gs), _lib.ptr(self.bcount), st),
                   "boundary")
        dist.all_reduce(self.bcount[s:e], op=dist.ReduceOp.SUM, group=self.group)
        self.comm_bytes += 4 * (e - s)
        nb_dev = self.scal[4:5]
        _lib.check(lib.vf_link_tables(C.byref(c), C.byref(gs), _lib.ptr(self.bcount),
                                      _lib.ptr(self.cmap), _lib.ptr(nb_dev), *self._ws("tables"), st),
                   "tables")
        _lib.check(lib.vf_check_status(C.byref(gs), st), "embed_geometry (sharded)")
        n_b = int(nb_dev.item())
        if self.lengths is None or self.lengths.shape[0] < n_b:
            cap = int(n_b * 1.25) + 16
            self.lengths = torch.empty((cap, 27, 64), dtype=torch.float32, device="cuda")
            self.bc_ids = torch.zeros((cap, 27, 64), dtype=torch.int8, device="cuda")
        lengths = self.lengths[:n_b]
        lengths.fill_(-1.0)
        lws = self.ws.get("links")
        need = lib.vf_link_workspace_size(C.byref(c), C.byref(gs))
        if lws is None or lws.numel() < need:
            lws = self.ws["links"] = torch.empty(int(need), dtype=torch.uint8, device="cuda")
        _lib.check(lib.vf_link_lengths(C.byref(c), C.byref(gs), _lib.ptr(self.cmap), faces, F, None,
                                       None, _lib.ptr(lengths), _lib.ptr(lws), lws.numel(), st),
                   "link lengths")
        return g, LinkTable(lengths, self.bc_ids[:n_b], self.cmap[:g.n_used], n_b)

    def owned_blocks(self, L: int):
        """Boolean (n_L,) ownership of the level-L blocks (ids in level order)."""
        s, e = self.grid.level_range(L)
        return self._owned(L, s, e)

    def cells_classified(self) -> int:
        return 64 * self.grid.n_used
