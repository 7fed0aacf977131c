"""voxelizer -- level-by-level solid voxelization, near-wall refinement,
boundary cells and the cut-link LUT on the GPU.

Drop-in for the SPEC ops of ``voxforest.voxelizer``:
  partial_surface_voxelize(grid, L, bins, mesh)   Alg. 3
  propagate_external(grid, L, direction)          Alg. 5
  finalize_masks(grid, L)
  mark_near_wall_refinement(grid, L, d_spec)
  identify_boundary_cells(grid)
  build_boundary_tables(grid)
  compute_link_lengths(grid, bins, mesh)
  (SPEC.md:328 / :337 signatures; the counts and the table may also be
  passed explicitly, else the grid carries them from the previous op)
  embed_geometry(grid, mesh, config)              SPEC.md:346-354 (native driver)
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import List, Optional, Tuple

from . import _lib, _ws
from .config import EmbedConfig
from .datatypes import BinLevel, ForestGrid, LinkTable, as_device_mesh


def _bins_struct(bins: BinLevel):
    b = bins._struct()
    return b


def partial_surface_voxelize(grid: ForestGrid, level: int, bins: BinLevel, mesh) -> ForestGrid:
    lib = _lib.require_cuda()
    dm = as_device_mesh(mesh)
    gs = grid._struct()
    c = _lib.make_config(grid.cfg)
    b = _bins_struct(bins)
    _lib.check(lib.vf_voxelize_level(C.byref(c), C.byref(gs), int(level), C.byref(b),
                                     _lib.ptr(dm.faces), _lib.stream_ptr()),
               "partial_surface_voxelize")
    return grid


def propagate_external(grid: ForestGrid, level: int, direction: int = +1,
                       finalize: bool = False) -> ForestGrid:
    """direction +1 = +x (all levels), -1 = -x (L > 0 only)."""
    lib = _lib.require_cuda()
    gs = grid._struct()
    c = _lib.make_config(grid.cfg)
    ws = _ws.get("propagate", lib.vf_propagate_workspace_size(C.byref(gs)))
    _lib.check(lib.vf_propagate_x(C.byref(c), C.byref(gs), int(level), int(direction),
                                  int(bool(finalize)), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
               "propagate_external")
    return grid


def finalize_masks(grid: ForestGrid, level: int) -> ForestGrid:
    lib = _lib.require_cuda()
    gs = grid._struct()
    c = _lib.make_config(grid.cfg)
    _lib.check(lib.vf_finalize_level(C.byref(c), C.byref(gs), int(level), _lib.stream_ptr()),
               "finalize_masks")
    return grid


def mark_near_wall_refinement(grid: ForestGrid, level: int, d_spec: Optional[float] = None):
    """Sets SB/SA/MARK block bits on level L; returns the level's mark mask."""
    lib = _lib.require_cuda()
    cfg = grid.cfg if d_spec is None else dataclasses.replace(grid.cfg, d_spec=float(d_spec))
    gs = grid._struct()
    c = _lib.make_config(cfg)
    ws = _ws.get("mark", lib.vf_mark_workspace_size(C.byref(gs)))
    _lib.check(lib.vf_mark_level(C.byref(c), C.byref(gs), int(level), _lib.ptr(ws), ws.numel(),
                                 _lib.stream_ptr()), "mark_near_wall_refinement")
    s, e = grid.level_range(level)
    return (grid.bflags[s:e] & _lib.BF_MARK) != 0


def identify_boundary_cells(grid: ForestGrid):
    """Finest level: FLUID cells with a SOLID same-level neighbour among the 26
    become BOUNDARY; returns per-block counts (capacity,) int32."""
    import torch
    lib = _lib.require_cuda()
    gs = grid._struct()
    c = _lib.make_config(grid.cfg)
    counts = torch.empty(grid.capacity, dtype=torch.int32, device="cuda")
    _lib.check(lib.vf_boundary_cells(C.byref(c), C.byref(gs), _lib.ptr(counts), _lib.stream_ptr()),
               "identify_boundary_cells")
    grid.bcount = counts
    return counts


def build_boundary_tables(grid: ForestGrid, counts=None) -> LinkTable:
    """contraction map (ascending block id) and LUT
    allocation, lengths = -1.  ``counts``: per-block boundary-cell counts;
    default: those of the grid's last identify_boundary_cells, else counted
    from the finest level's BOUNDARY cell masks."""
    import torch
    lib = _lib.require_cuda()
    if counts is None:
        counts = grid.bcount
    if counts is None:
        counts = torch.zeros(grid.capacity, dtype=torch.int32, device="cuda")
        s, e = grid.level_range(grid.n_levels - 1)
        counts[s:e] = (grid.masks[s:e] == _lib.BOUNDARY).sum(dim=1, dtype=torch.int32)
    gs = grid._struct()
    c = _lib.make_config(grid.cfg)
    cmap = torch.empty(grid.capacity, dtype=torch.int32, device="cuda")
    nb = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = _ws.get("tables", lib.vf_tables_workspace_size(C.byref(gs)))
    _lib.check(lib.vf_link_tables(C.byref(c), C.byref(gs), _lib.ptr(counts), _lib.ptr(cmap),
                                  _lib.ptr(nb), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
               "build_boundary_tables")
    n_b = int(nb.item())
    lengths = torch.full((n_b, 27, 64), -1.0, dtype=torch.float32, device="cuda")
    bc_ids = torch.zeros((n_b, 27, 64), dtype=torch.int8, device="cuda")
    grid.table = LinkTable(lengths, bc_ids, cmap[:grid.n_used], n_b)
    return grid.table


def compute_link_lengths(grid: ForestGrid, bins: Optional[BinLevel], mesh,
                         table: Optional[LinkTable] = None) -> LinkTable:
    """fill the LUT with q = d/dx in (0, 1] (min over faces)
    for every cell of every mapped block and q = 1..26; -1 where no wall is
    within one link.  ``table``: default the grid's last
    build_boundary_tables.  ``bins`` (all-directions BinLevel) only restricts
    the face set via its filter map; the result is invariant to it
    (SPEC.md:174)."""
    lib = _lib.require_cuda()
    if table is None:
        table = grid.table
    if table is None:
        raise ValueError("compute_link_lengths: no LinkTable (call build_boundary_tables first)")
    dm = as_device_mesh(mesh)
    gs = grid._struct()
    c = _lib.make_config(grid.cfg)
    ws = _ws.get("links", lib.vf_link_workspace_size(C.byref(c), C.byref(gs)))
    fmap = n_map = None
    keep = []
    if bins is not None and bins.filter_map is not None:
        import torch
        fmap = bins.filter_map.compact_map.to(torch.int32).contiguous()
        n_map = torch.tensor([fmap.numel()], dtype=torch.int32, device="cuda")
        keep = [fmap, n_map]
    cmap_full = table.contraction_map
    if cmap_full.numel() < grid.capacity:
        import torch
        full = torch.full((grid.capacity,), -1, dtype=torch.int32, device="cuda")
        full[:cmap_full.numel()] = cmap_full
        cmap_full = full
    _lib.check(lib.vf_link_lengths(C.byref(c), C.byref(gs), _lib.ptr(cmap_full), _lib.ptr(dm.faces),
                                   dm.n_faces, _lib.ptr(fmap), _lib.ptr(n_map),
                                   _lib.ptr(table.lengths), _lib.ptr(ws), ws.numel(),
                                   _lib.stream_ptr()), "compute_link_lengths")
    del keep
    return table


# ---------------------------------------------------------------------------
# embed_geometry: one native driver call per phase, no host sync inside a level

@dataclasses.dataclass
class EmbedTimings:
    """Per-stage device times (ms) grouped like the paper's table
    (PAPER.md:1052-1080 / SPEC.md:498)."""
    binning: float = 0.0
    voxelization: float = 0.0
    refinement: float = 0.0
    boundary: float = 0.0
    links: float = 0.0
    total: float = 0.0


class EmbedEngine:
    """Reusable embed context for one (mesh, cfg): device mesh, forest arrays,
    workspace, LUT and -- after the first run -- a CUDA graph of the whole
    embed are allocated once and reused (the geometry is static,
    PAPER.md:273).  All work runs on the engine's own stream, ordered after
    the caller's current stream."""

    # above this many faces the embed is throughput-bound: eager launches keep
    # the stream priorities (the low-priority cut-link enumeration yields to
    # the level pipeline), which CUDA-graph node priorities did not reproduce
    # (C4: 5.0 ms eager vs 5.6 ms graph); below it the graph saves launches
    GRAPH_MAX_FACES = 1_000_000

    def __init__(self, mesh, cfg: EmbedConfig, capacity: Optional[int] = None,
                 use_graph: Optional[bool] = None):
        import torch
        self.lib = _lib.require_cuda()
        self.cfg = cfg
        self.mesh = as_device_mesh(mesh)
        cap = int(capacity if capacity is not None else cfg.block_capacity(self.mesh.area))
        self.grid = ForestGrid.allocate(cfg, cap)
        self.c = _lib.make_config(cfg)
        # cut-link line records: ~9 piercing lines per finest cell area of
        # surface over the 13 direction pairs (measured on the torus meshes);
        # re-sized after the first run if they overflow
        dxf = cfg.dx(cfg.l_max - 1)
        self.c.line_cap = max(2 * self.mesh.n_faces, int(12 * self.mesh.area / (dxf * dxf)), 1 << 22)
        wsb = self.lib.vf_embed_workspace_size(C.byref(self.c), self.mesh.n_faces, cap)
        if wsb == 0:
            raise ValueError("invalid embed configuration")
        self.ws = torch.empty(int(wsb), dtype=torch.uint8, device="cuda")
        self.cmap = torch.empty(cap, dtype=torch.int32, device="cuda")
        self.n_b_dev = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.host = torch.zeros(8, dtype=torch.int32).pin_memory()  # 0-3 status, 4 n_b
        # the level pipeline is the critical path: above the library's bins
        # stream (-1) and its low-priority cut-link enumeration (0), below its
        # next-level row order (-3)
        self.stream = torch.cuda.Stream(priority=-2)
        self.lengths = None
        self.bc_ids = None
        self.lengths_cap = 0
        self.use_graph = (self.mesh.n_faces <= self.GRAPH_MAX_FACES) if use_graph is None else use_graph
        self._graphs = {}
        self.n_events = 64
        self.events = [torch.cuda.Event(enable_timing=True) for _ in range(self.n_events)]
        self._ev_arr = None

    def __del__(self):
        try:
            for g in self._graphs.values():
                self.lib.vf_graph_destroy(g)
        except Exception:
            pass

    def _ensure_events(self):
        if self._ev_arr is None:
            for e in self.events:   # handles are created lazily on first record
                e.record(self.stream)
            self._ev_arr = (C.c_void_p * self.n_events)(*[C.c_void_p(e.cuda_event) for e in self.events])

    def _alloc_lut(self, n_b: int):
        import torch
        cap = int(n_b * 1.25) + 16
        self.lengths = torch.empty((cap, 27, 64), dtype=torch.float32, device="cuda")
        self.bc_ids = torch.zeros((cap, 27, 64), dtype=torch.int8, device="cuda")
        self.lengths_cap = cap
        for g in self._graphs.values():
            self.lib.vf_graph_destroy(g)
        self._graphs.clear()

    def _phase1(self, uf, st, ev):
        gs = self.grid._struct()
        _lib.check(self.lib.vf_embed_phase1(
            C.byref(self.c), _lib.ptr(self.mesh.faces), self.mesh.n_faces, int(bool(uf)), C.byref(gs),
            _lib.ptr(self.cmap), _lib.ptr(self.n_b_dev), _lib.ptr(self.ws), self.ws.numel(), st, ev),
            "embed_geometry")
        self.grid.n_levels = gs.n_levels
        return gs

    def _phase2(self, gs, st, lev):
        _lib.check(self.lib.vf_embed_phase2(
            C.byref(self.c), _lib.ptr(self.mesh.faces), self.mesh.n_faces, C.byref(gs),
            _lib.ptr(self.cmap), _lib.ptr(self.n_b_dev), _lib.ptr(self.lengths), self.lengths_cap,
            _lib.ptr(self.ws), self.ws.numel(), st, lev), "embed_geometry")

    def _grow_pairs(self) -> bool:
        """After a phase 1: if the per-level (bin, face) pair list overflowed
        (VF_ECAPACITY with the required count in status[3]), enlarge it and
        the workspace; True = rerun."""
        import torch
        self.host[0:4].copy_(self.grid.status, non_blocking=True)
        self.stream.synchronize()
        _lib.check(self.lib.vf_side_sync(), "embed_geometry")
        need = int(self.host[3])
        if int(self.host[0]) != 2 or need <= 0:
            return False
        self.c.pair_cap = int(need * 1.25) + 65536
        self._realloc_ws()
        return True

    def _grow_lines(self) -> bool:
        """After a phase 1: if the cut-link line records or the band list
        overflowed (correct, but redone by the slow exact kernels), enlarge
        them and the workspace; True = rerun."""
        st = self.link_stats()
        need = max(st["lines"], 16 * st["band"])
        if need <= st["line_cap"] and st["band"] <= st["band_cap"]:
            return False
        self.c.line_cap = int(need * 1.25) + 65536
        self._realloc_ws()
        return True

    def _realloc_ws(self):
        import torch
        wsb = self.lib.vf_embed_workspace_size(C.byref(self.c), self.mesh.n_faces, self.grid.capacity)
        self.ws = None
        self.ws = torch.empty(int(wsb), dtype=torch.uint8, device="cuda")
        for g in self._graphs.values():
            self.lib.vf_graph_destroy(g)
        self._graphs.clear()

    def _finish(self, st_obj):
        """Async read of status + N_b, one sync, error mapping."""
        import torch
        self.host[0:4].copy_(self.grid.status, non_blocking=True)
        self.host[4:5].copy_(self.n_b_dev, non_blocking=True)
        st_obj.synchronize()
        # the side streams (cut-link enumeration) are done after phase 2; after
        # a phase 1 alone (LUT sizing, errors) wait for them explicitly
        _lib.check(self.lib.vf_side_sync(), "embed_geometry")
        h = self.host.tolist()
        if h[0]:
            gs = self.grid._struct()
            _lib.check(self.lib.vf_check_status(C.byref(gs), _lib.stream_ptr(st_obj)), "embed_geometry")
        return int(h[4])

    def run(self, timed: bool = False, use_filter: Optional[bool] = None):
        """Full embed -> (grid, LinkTable).  Steady state is one CUDA-graph
        launch and one host sync at the end (status + N_b)."""
        import torch
        uf = bool(self.cfg.use_filter if use_filter is None else use_filter)
        cur = torch.cuda.current_stream()
        self.stream.wait_stream(cur)
        st = _lib.stream_ptr(self.stream)
        with torch.cuda.stream(self.stream):
            if self.lengths is None:
                # first run: learn N_b (one extra sync), size the LUT; a
                # (bin, face) pair list that overflowed is re-sized and rerun
                while True:
                    self.grid.status.zero_()
                    gs = self._phase1(uf, st, None)
                    if self._grow_pairs():
                        continue
                    n_b = self._finish(self.stream)
                    if self._grow_lines():
                        continue
                    break
                self._alloc_lut(n_b)
            if timed or not self.use_graph:
                self._ensure_events()
                self.grid.status.zero_()
                ev = C.cast(self._ev_arr, C.POINTER(C.c_void_p)) if timed else None
                gs = self._phase1(uf, st, ev)
                lev = (C.cast(C.byref(self._ev_arr, C.sizeof(C.c_void_p) * (self.n_events - 3)),
                              C.POINTER(C.c_void_p)) if timed else None)
                self._phase2(gs, st, lev)
                if timed:
                    self.events[self.n_events - 1].record(self.stream)
            else:
                g = self._graphs.get(uf)
                if g is None:
                    gs = self.grid._struct()
                    h = C.c_void_p()
                    _lib.check(self.lib.vf_embed_graph_create(
                        C.byref(self.c), _lib.ptr(self.mesh.faces), self.mesh.n_faces, int(uf),
                        C.byref(gs), _lib.ptr(self.cmap), _lib.ptr(self.n_b_dev),
                        _lib.ptr(self.lengths), self.lengths_cap, _lib.ptr(self.ws), self.ws.numel(),
                        st, C.byref(h)), "embed_geometry (graph capture)")
                    g = self._graphs[uf] = h.value
                self.grid.status.zero_()
                _lib.check(self.lib.vf_graph_launch(g, st), "embed_geometry")
                self.grid.n_levels = self.cfg.l_max
            n_b = self._finish(self.stream)
            if self.host[0].item() == 0 and n_b > self.lengths_cap:  # defensive
                self._alloc_lut(n_b)
                return self.run(timed, use_filter)
        cur.wait_stream(self.stream)
        self._n_used = int(self.grid.level_start[self.grid.n_levels].item())  # static for a fixed mesh
        table = LinkTable(self.lengths[:n_b], self.bc_ids[:n_b], self.cmap, n_b)
        return self.grid, table

    # -- pipelined serving path ---------------------------------------------
    def run_async(self, use_filter: Optional[bool] = None):
        """Enqueue one embed on the engine stream without a host sync (steady
        state: the LUT is sized, N_b is static for a fixed mesh).  The status
        and N_b are copied back asynchronously; check_async() validates them."""
        import torch
        if self.lengths is None:
            return self.run(use_filter=use_filter)
        uf = bool(self.cfg.use_filter if use_filter is None else use_filter)
        st = _lib.stream_ptr(self.stream)
        n_b = int(self.host[4])
        with torch.cuda.stream(self.stream):
            self.grid.status.zero_()
            if self.use_graph and uf in self._graphs:
                _lib.check(self.lib.vf_graph_launch(self._graphs[uf], st), "embed_geometry")
            else:
                gs = self._phase1(uf, st, None)
                self._phase2(gs, st, None)
            self.grid.n_levels = self.cfg.l_max
            if not hasattr(self, "_host_async"):
                self._host_async = torch.zeros(8, dtype=torch.int32).pin_memory()
            self._host_async[0:4].copy_(self.grid.status, non_blocking=True)
            self._host_async[4:5].copy_(self.n_b_dev, non_blocking=True)
            L = self.cfg.l_max
            self._host_async[5:6].copy_(self.grid.level_start[L:L + 1], non_blocking=True)
        table = LinkTable(self.lengths[:n_b], self.bc_ids[:n_b], self.cmap, n_b)
        return self.grid, table

    def check_async(self):
        """Validate the last run_async (synchronizes the engine stream)."""
        self.stream.synchronize()
        h = self._host_async.tolist() if hasattr(self, "_host_async") else self.host.tolist()
        indexed = getattr(self, "_indexed_pending", False)
        self._indexed_pending = False
        if indexed and h[7]:      # the uploaded mesh was invalid: nothing else is meaningful
            _lib.check(int(h[7]), "pack_indexed (invalid mesh)")
        if h[0]:
            gs = self.grid._struct()
            _lib.check(self.lib.vf_check_status(C.byref(gs), _lib.stream_ptr(self.stream)), "embed_geometry")
        if h[4] != int(self.host[4]):
            raise RuntimeError("N_b changed between pipelined embeds of the same mesh")
        if hasattr(self, "_host_async") and h[5] != self._n_used:
            raise RuntimeError("the block count changed between pipelined embeds: the downloaded "
                               "grid slices were sized by the previous synchronous run")
        if indexed:
            if h[6] != self._n_links:
                raise RuntimeError("the cut-link count changed between pipelined embeds of the same mesh")

    def embed_host_async(self, faces_coord, normals, out, in_stream, out_stream):
        """One pipelined end-to-end step: pinned host faces -> H2D on
        ``in_stream`` -> pack + embed on the engine stream -> D2H of the
        results on ``out_stream`` into the pinned ``out`` buffers (allocated on
        first use).  No host sync: with two engines alternating, the D2H of one
        step overlaps the next step's upload and compute.  Returns (out, h2d
        bytes, d2h bytes)."""
        import torch
        F = self.mesh.n_faces
        if not hasattr(self, "_dfc"):
            self._dfc = torch.empty((F, 9), dtype=torch.float64, device="cuda")
            self._dn = torch.empty((F, 3), dtype=torch.float64, device="cuda")
            self._ev_pack = torch.cuda.Event()
            self._ev_h2d = torch.cuda.Event()
            self._ev_done = torch.cuda.Event()
            self._ev_d2h = torch.cuda.Event()
            self._ev_pack.record(self.stream)
            self._ev_d2h.record(out_stream)
        in_stream.wait_event(self._ev_pack)        # the previous pack has read the buffers
        with torch.cuda.stream(in_stream):
            self._dfc.copy_(faces_coord, non_blocking=True)
            self._dn.copy_(normals, non_blocking=True)
            self._ev_h2d.record(in_stream)
        self.stream.wait_event(self._ev_h2d)
        self.stream.wait_event(self._ev_d2h)       # the previous results were copied out
        _lib.check(self.lib.vf_pack_faces(_lib.ptr(self._dfc), _lib.ptr(self._dn), F,
                                          _lib.ptr(self.mesh.faces), _lib.stream_ptr(self.stream)),
                   "pack_faces")
        self._ev_pack.record(self.stream)
        grid, table = self.run_async()
        self._ev_done.record(self.stream)
        out_stream.wait_event(self._ev_done)
        n = self._n_used  # from the last synchronous run (no host sync here)
        res = {"coords": grid.coords[:n], "nbr": grid.nbr[:n], "child": grid.child[:n],
               "bflags": grid.bflags[:n], "masks": grid.masks[:n],
               "contraction_map": table.contraction_map[:n], "lengths": table.lengths}
        if out is None:
            out = {}
        d2h = 0
        with torch.cuda.stream(out_stream):
            for k, t in res.items():
                buf = out.get(k)
                if buf is None or buf.shape != t.shape:
                    buf = torch.empty(t.shape, dtype=t.dtype).pin_memory()
                    out[k] = buf
                buf.copy_(t, non_blocking=True)
                d2h += t.numel() * t.element_size()
            self._ev_d2h.record(out_stream)
        h2d = faces_coord.numel() * 8 + normals.numel() * 8
        return out, h2d, d2h

    def _indexed_setup(self, V: int, F: int):
        """Device buffers of the indexed serving path; sizes the sparse LUT
        download from the current LUT (one sync, outside any timed step)."""
        import torch
        self._dverts = torch.empty((V, 3), dtype=torch.float64, device="cuda")
        self._dfidx = torch.empty((F, 3), dtype=torch.int32, device="cuda")
        self._pack_status = torch.zeros(4, dtype=torch.int32, device="cuda")
        self._sp_count = torch.zeros(1, dtype=torch.int32, device="cuda")
        self._sp_ws = torch.empty(int(self.lib.vf_lut_sparse_workspace_size(self.lengths_cap)), dtype=torch.uint8,
                                  device="cuda")
        dummy = torch.empty(1, dtype=torch.int32, device="cuda")
        _lib.check(self.lib.vf_lut_sparse(_lib.ptr(self.lengths), self.lengths_cap, _lib.ptr(self.n_b_dev),
                                          _lib.ptr(dummy), _lib.ptr(dummy), 0, _lib.ptr(self._sp_count),
                                          _lib.ptr(self._sp_ws), self._sp_ws.numel(), _lib.stream_ptr(self.stream)),
                   "lut_sparse")
        self.stream.synchronize()
        self._n_links = int(self._sp_count.item())
        cap = self._n_links + 1024
        self._sp_idx = torch.empty(cap, dtype=torch.int32, device="cuda")
        self._sp_val = torch.empty(cap, dtype=torch.float32, device="cuda")
        self._ev_sp = torch.cuda.Event()

    def embed_indexed_async(self, vertices, faces_idx, out, in_stream, out_stream):
        """One pipelined end-to-end step from the reference mesh's own fields:
        pinned host ``vertices`` (V,3) f64 and ``faces_idx`` (F,3) int32 ->
        H2D on ``in_stream`` (24 B/vertex + 12 B/face) -> face records and
        unit normals on the device (vf_pack_indexed, TriangleMesh's
        np.cross / norm bit for bit) -> embed -> the cut links of the LUT as
        (flat index, q) pairs (vf_lut_sparse) -> D2H on ``out_stream`` of the
        grid (coords, nbr, child, bflags, masks, contraction map) and the
        sparse LUT into pinned ``out`` buffers.  No host sync; check_async()
        validates the step.  Returns (out, h2d bytes, d2h bytes)."""
        import torch
        V, F = int(vertices.shape[0]), int(faces_idx.shape[0])
        if F != self.mesh.n_faces:
            raise ValueError("embed_indexed_async: face count differs from the engine's mesh")
        if self.lengths is None:
            self.run()
        if not hasattr(self, "_dfidx") or self._dverts.shape[0] != V:
            self._indexed_setup(V, F)
            self._ev_pack = torch.cuda.Event()
            self._ev_h2d = torch.cuda.Event()
            self._ev_done = torch.cuda.Event()
            self._ev_d2h = torch.cuda.Event()
            self._ev_pack.record(self.stream)
            self._ev_d2h.record(out_stream)
        in_stream.wait_event(self._ev_pack)        # the previous pack has read the buffers
        with torch.cuda.stream(in_stream):
            self._dverts.copy_(vertices, non_blocking=True)
            self._dfidx.copy_(faces_idx, non_blocking=True)
            self._ev_h2d.record(in_stream)
        self.stream.wait_event(self._ev_h2d)
        self.stream.wait_event(self._ev_d2h)       # the previous results were copied out
        st = _lib.stream_ptr(self.stream)
        _lib.check(self.lib.vf_pack_indexed(_lib.ptr(self._dverts), V, _lib.ptr(self._dfidx), F,
                                            _lib.ptr(self.mesh.faces), _lib.ptr(self._pack_status), st),
                   "pack_indexed")
        self._ev_pack.record(self.stream)
        grid, table = self.run_async()
        _lib.check(self.lib.vf_lut_sparse(_lib.ptr(self.lengths), self.lengths_cap, _lib.ptr(self.n_b_dev),
                                          _lib.ptr(self._sp_idx), _lib.ptr(self._sp_val), self._sp_idx.numel(),
                                          _lib.ptr(self._sp_count), _lib.ptr(self._sp_ws), self._sp_ws.numel(), st),
                   "lut_sparse")
        with torch.cuda.stream(self.stream):
            self._host_async[6:7].copy_(self._sp_count, non_blocking=True)
            self._host_async[7:8].copy_(self._pack_status[0:1], non_blocking=True)
        self._ev_done.record(self.stream)
        out_stream.wait_event(self._ev_done)
        n, k = self._n_used, self._n_links
        res = {"coords": grid.coords[:n], "nbr": grid.nbr[:n], "child": grid.child[:n],
               "bflags": grid.bflags[:n], "masks": grid.masks[:n],
               "contraction_map": table.contraction_map[:n], "link_index": self._sp_idx[:k],
               "link_q": self._sp_val[:k]}
        if out is None:
            out = {}
        d2h = 0
        # the download in two concurrent copies (~half the bytes each: the
        # neighbour rows, link indices and child ids beside the rest; measured
        # ~2-3% more PCIe throughput than one stream), joined on out_stream
        if not hasattr(self, "_out2"):
            self._out2 = torch.cuda.Stream()
            self._ev_out2 = torch.cuda.Event()
        self._out2.wait_event(self._ev_done)
        with torch.cuda.stream(out_stream):
            for key, t in res.items():
                buf = out.get(key)
                if buf is None or buf.shape != t.shape:
                    buf = torch.empty(t.shape, dtype=t.dtype).pin_memory()
                    out[key] = buf
                if key in ("nbr", "link_index", "child"):
                    with torch.cuda.stream(self._out2):
                        buf.copy_(t, non_blocking=True)
                else:
                    buf.copy_(t, non_blocking=True)
                d2h += t.numel() * t.element_size()
            self._ev_out2.record(self._out2)
            out_stream.wait_event(self._ev_out2)
            self._ev_d2h.record(out_stream)
        self._indexed_pending = True
        return out, V * 24 + F * 12, d2h

    @property
    def n_b_host(self):
        return self.host[4:5]

    def timings(self) -> EmbedTimings:
        """Stage split of the last timed run (call after synchronize)."""
        ev = self.events
        L = self.cfg.l_max
        t = EmbedTimings()
        k = 0
        for lv in range(L):
            t.binning += ev[k].elapsed_time(ev[k + 1])
            t.voxelization += ev[k + 1].elapsed_time(ev[k + 2])
            k += 2
            if lv < L - 1:
                t.refinement += ev[k].elapsed_time(ev[k + 1])
                k += 1
        t.boundary = ev[k].elapsed_time(ev[k + 1])
        t.links = ev[k + 1].elapsed_time(ev[self.n_events - 1])
        t.total = ev[0].elapsed_time(ev[self.n_events - 1])
        return t

    def kernel_times(self, gate_us: float = 3000.0, use_filter: Optional[bool] = None) -> dict:
        """Per-kernel device times of one eager embed with every kernel on
        the engine stream in order (vf_ktimer_*): {name: (launches, total
        ms)}.  Attribution only -- the production schedule overlaps the bins
        and the cut-link enumeration with the level pipeline."""
        import torch
        if self.lengths is None:
            self.run()
        uf = bool(self.cfg.use_filter if use_filter is None else use_filter)
        st = _lib.stream_ptr(self.stream)
        torch.cuda.synchronize()
        _lib.check(self.lib.vf_ktimer_start(st, float(gate_us)), "kernel_times")
        try:
            with torch.cuda.stream(self.stream):
                self.grid.status.zero_()
                gs = self._phase1(uf, st, None)
                self._phase2(gs, st, None)
        finally:
            buf = C.create_string_buffer(1 << 16)
            n = self.lib.vf_ktimer_stop(buf, len(buf))
        if n < 0:
            _lib.check(-n, "kernel_times")
        self._finish(self.stream)
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ms = line.split("\t")
            out[name] = (int(cnt), float(ms))
        return out

    def link_stats(self) -> dict:
        """Counters of the last embed's cut-link pass (synchronises): lines
        recorded by the enumeration and the buffer capacity, faces whose lines
        overflowed it (redone by the direct kernel), band candidates (exact
        SAT path), the band capacity, the faces of the large-face kernel and
        the lattice lines the enumeration classified (FP32 intersection tests)."""
        import torch
        torch.cuda.current_stream().synchronize()
        self.lib.vf_side_sync()
        out = (C.c_int64 * 7)()
        _lib.check(self.lib.vf_embed_link_stats(C.byref(self.c), self.mesh.n_faces, self.grid.capacity,
                                                _lib.ptr(self.ws), self.ws.numel(), out), "link_stats")
        return dict(zip(("lines", "line_cap", "overflow_faces", "band", "band_cap", "large_faces", "tests"),
                        map(int, out)))

    def link_kernel_ms(self) -> float:
        """Device time of the cut-link kernels of the last timed run: the line
        enumeration (side stream, overlapped with the level pipeline, events
        58-59) plus the LUT fill and the resolution after the tables (events
        61-62)."""
        enum = self.events[58].elapsed_time(self.events[59])
        return enum + self.events[self.n_events - 3].elapsed_time(self.events[self.n_events - 2])

    def link_enum_ms(self) -> float:
        """The overlapped part of link_kernel_ms (grid-independent enumeration)."""
        return self.events[58].elapsed_time(self.events[59])

    def cells_classified(self) -> int:
        """Sum over levels of 64 * blocks."""
        return 64 * self.grid.n_used

    # -- end-to-end path: host mesh in, host results out -------------------
    def embed_host(self, faces_coord, normals, out=None):
        """Upload host face arrays (pinned for async copies), embed, and copy
        the results back into pinned host buffers ``out`` (allocated on first
        use).  Returns (out, h2d_bytes, d2h_bytes)."""
        import torch
        lib = self.lib
        F = self.mesh.n_faces
        if not hasattr(self, "_dfc"):
            self._dfc = torch.empty((F, 9), dtype=torch.float64, device="cuda")
            self._dn = torch.empty((F, 3), dtype=torch.float64, device="cuda")
        self._dfc.copy_(faces_coord, non_blocking=True)
        self._dn.copy_(normals, non_blocking=True)
        _lib.check(lib.vf_pack_faces(_lib.ptr(self._dfc), _lib.ptr(self._dn), F,
                                     _lib.ptr(self.mesh.faces), _lib.stream_ptr()), "pack_faces")
        grid, table = self.run()
        n = grid.n_used
        res = {"coords": grid.coords[:n], "nbr": grid.nbr[:n], "child": grid.child[:n],
               "bflags": grid.bflags[:n], "masks": grid.masks[:n],
               "contraction_map": table.contraction_map[:n], "lengths": table.lengths}
        if out is None:
            out = {}
        d2h = 0
        for k, t in res.items():
            buf = out.get(k)
            if buf is None or buf.shape != t.shape:
                buf = torch.empty(t.shape, dtype=t.dtype).pin_memory()
                out[k] = buf
            buf.copy_(t, non_blocking=True)
            d2h += t.numel() * t.element_size()
        h2d = faces_coord.numel() * 8 + normals.numel() * 8
        return out, h2d, d2h


_ENGINES: "collections.OrderedDict" = None
_ENGINE_CACHE = 4


def _mesh_key(mesh):
    """Identity of a mesh's geometry: the face/normal arrays (object and
    buffer address) -- a TriangleMesh is immutable (geometry.py:65-111)."""
    import weakref
    fc, nrm = mesh.faces_coord, mesh.normals
    try:
        ref = weakref.ref(mesh)
    except TypeError:
        ref = None
    addr = lambda a: a.ctypes.data if hasattr(a, "ctypes") else (a.data_ptr() if hasattr(a, "data_ptr") else id(a))
    return (id(mesh), id(fc), addr(fc), id(nrm), addr(nrm), tuple(getattr(fc, "shape", ()))), ref


def embed_geometry(grid: Optional[ForestGrid], mesh, cfg: EmbedConfig,
                   capacity: Optional[int] = None, copy: bool = False) -> Tuple[ForestGrid, LinkTable]:
    """build the forest level by level around the mesh and
    return (grid, LinkTable).  ``grid`` may be a fresh root grid from
    init_forest (its capacity is reused) or None.

    The EmbedEngine (device mesh, forest arrays, workspace, LUT, CUDA graph)
    is cached per (mesh geometry, cfg, capacity), up to 4 engines: a repeated
    call is one graph launch.  The returned grid / table are that engine's
    buffers and are overwritten by the next call with the same key; pass
    ``copy=True`` for independent copies."""
    import collections
    global _ENGINES
    if grid is not None and capacity is None:
        capacity = grid.capacity
    if _ENGINES is None:
        _ENGINES = collections.OrderedDict()
    mk, ref = _mesh_key(mesh)
    key = (mk, cfg, capacity)
    hit = _ENGINES.get(key)
    eng = None
    if hit is not None:
        eng, r = hit
        if r is not None and r() is not mesh:   # id reused by another object
            eng = None
    if eng is None:
        eng = EmbedEngine(mesh, cfg, capacity)
        _ENGINES[key] = (eng, ref)
        while len(_ENGINES) > _ENGINE_CACHE:
            _ENGINES.popitem(last=False)
    else:
        _ENGINES.move_to_end(key)
    g, t = eng.run()
    if copy:
        g = dataclasses.replace(g, **{f.name: getattr(g, f.name).clone() for f in dataclasses.fields(g)
                                      if hasattr(getattr(g, f.name), "clone")})
        t = LinkTable(t.lengths.clone(), t.bc_ids.clone(), t.contraction_map.clone(), t.n_b)
    return g, t
