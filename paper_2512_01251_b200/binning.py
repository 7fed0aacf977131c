"""binning -- spatial-bin hierarchy on the GPU.

Drop-in for the reference SPEC ops ``voxforest.binning.*`` (the reference
module is specification-only).  Each op is
one call into libvoxforest_b200.so; outputs are torch CUDA tensors.

  compute_ray_indicators(mesh, level, mode)   SPEC.md:124-132, Alg. 1
  compact_filtered_faces(indicators)
  compute_bin_pairs(mesh, filter, level)      SPEC.md:142-150, Alg. 2
  assemble_bins(pairs, n_bins)                SPEC.md:151-159, steps 3-9
  build_bin_hierarchy(mesh, config)
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Tuple

from . import _lib, _ws
from .config import EmbedConfig
from .datatypes import BinLevel, FilterMap, as_device_mesh

AXIS_ONLY = "axis-only"
ALL_DIRECTIONS = "all-directions"


def _mode(mode) -> int:
    if mode in (0, "axis", AXIS_ONLY, "1d", "1D"):
        return 0
    if mode in (1, "all", ALL_DIRECTIONS, "md", "MD"):
        return 1
    raise ValueError(f"unknown indicator mode {mode!r}")


def compute_ray_indicators(mesh, level: int, mode=AXIS_ONLY, cfg: EmbedConfig = EmbedConfig()):
    """Per-face 0/1: some level-L lattice ray (x rows, or the 13 antiparallel
    direction pairs in all-directions mode) pierces the face."""
    import torch
    lib = _lib.require_cuda()
    dm = as_device_mesh(mesh)
    out = torch.empty(dm.n_faces, dtype=torch.uint8, device="cuda")
    c = _lib.make_config(cfg)
    _lib.check(lib.vf_ray_indicators(C.byref(c), _lib.ptr(dm.faces), dm.n_faces, int(level),
                                     _mode(mode), _lib.ptr(out), _lib.stream_ptr()),
               "compute_ray_indicators")
    return out


def compact_filtered_faces(indicators) -> FilterMap:
    """Ascending original ids of faces with indicator 1."""
    import torch
    lib = _lib.require_cuda()
    ind = indicators.to(device="cuda", dtype=torch.uint8).contiguous()
    n = ind.numel()
    cmap = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = _ws.get("compact", lib.vf_compact_workspace_size(n))
    _lib.check(lib.vf_compact(_lib.ptr(ind), n, _lib.ptr(cmap), _lib.ptr(cnt), _lib.ptr(ws),
                              ws.numel(), _lib.stream_ptr()), "compact_filtered_faces")
    k = int(cnt.item())
    return FilterMap(ind, cmap[:k])


def compute_bin_pairs(mesh, fmap: Optional[FilterMap], level: int,
                      cfg: EmbedConfig = EmbedConfig()) -> Tuple[object, object]:
    """(bin, face) pairs of Alg. 2 in face-major emission order; raises
    BinCapError when a face exceeds N_lim = (2+N_spec)^3."""
    import torch
    lib = _lib.require_cuda()
    dm = as_device_mesh(mesh)
    c = _lib.make_config(cfg)
    if fmap is None:
        fmap_t, n_map = None, dm.n_faces
    else:
        fmap_t = fmap.compact_map.to(device="cuda", dtype=torch.int32).contiguous()
        n_map = fmap_t.numel()
    cap = max(n_map * cfg.n_lim, 1)
    pb = torch.empty(cap, dtype=torch.int32, device="cuda")
    pf = torch.empty(cap, dtype=torch.int32, device="cuda")
    scal = torch.zeros(4, dtype=torch.int32, device="cuda")  # 0 n_pairs, 1 status, 2 n_map
    scal[2] = n_map
    wsb = lib.vf_bins_workspace_size(C.byref(c), dm.n_faces, int(level))
    ws = _ws.get("bins", wsb)
    _lib.check(lib.vf_bin_pairs(C.byref(c), _lib.ptr(dm.faces), dm.n_faces,
                                _lib.ptr(fmap_t) if fmap_t is not None else None,
                                C.c_void_p(scal.data_ptr() + 8) if fmap_t is not None else None,
                                int(level), _lib.ptr(pb), _lib.ptr(pf), cap,
                                _lib.ptr(scal), C.c_void_p(scal.data_ptr() + 4), _lib.ptr(ws),
                                ws.numel(), _lib.stream_ptr()), "compute_bin_pairs")
    h = scal.cpu().numpy()
    if h[1]:
        _lib.check(int(h[1]), "compute_bin_pairs")
    n = int(h[0])
    return pb[:n], pf[:n]


def assemble_bins(pairs, n_bins: int, level: int = 0, bin_density=None) -> BinLevel:
    """Group pairs by bin: counts, offsets, face_ids ascending within a bin
    (stable key sort)."""
    import torch
    lib = _lib.require_cuda()
    pb, pf = pairs
    pb = pb.to(device="cuda", dtype=torch.int32).contiguous()
    pf = pf.to(device="cuda", dtype=torch.int32).contiguous()
    P = pb.numel()
    counts = torch.empty(int(n_bins), dtype=torch.int32, device="cuda")
    offsets = torch.empty(int(n_bins), dtype=torch.int32, device="cuda")
    face_ids = torch.empty(max(P, 1), dtype=torch.int32, device="cuda")
    npairs = torch.tensor([P], dtype=torch.int32, device="cuda")
    ws = _ws.get("assemble", lib.vf_assemble_workspace_size(max(P, 1), int(n_bins)))
    _lib.check(lib.vf_bin_assemble(_lib.ptr(pb), _lib.ptr(pf), _lib.ptr(npairs), max(P, 1),
                                   int(n_bins), _lib.ptr(counts), _lib.ptr(offsets),
                                   _lib.ptr(face_ids), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
               "assemble_bins")
    if bin_density is None:
        b = round(int(n_bins) ** (1.0 / 3.0))
        bin_density = (b, b, b)
    return BinLevel(level, tuple(bin_density), face_ids[:P], counts, offsets)


def build_level(mesh, level: int, cfg: EmbedConfig = EmbedConfig(), mode=AXIS_ONLY,
                use_filter: Optional[bool] = None) -> BinLevel:
    """Fused one-level build (indicators -> compact -> pairs -> counting sort)."""
    import torch
    lib = _lib.require_cuda()
    dm = as_device_mesh(mesh)
    c = _lib.make_config(cfg)
    nb = cfg.n_bins(level)
    F = dm.n_faces
    cap = F * cfg.n_lim
    counts = torch.empty(nb, dtype=torch.int32, device="cuda")
    offsets = torch.empty(nb, dtype=torch.int32, device="cuda")
    face_ids = torch.empty(cap, dtype=torch.int32, device="cuda")
    fmap = torch.empty(F, dtype=torch.int32, device="cuda")
    scal = torch.zeros(4, dtype=torch.int32, device="cuda")  # 0 n_face_ids, 1 n_map, 2 status
    b = _lib.VfBins()
    b.d_counts, b.d_offsets, b.d_face_ids = counts.data_ptr(), offsets.data_ptr(), face_ids.data_ptr()
    b.face_ids_cap = cap
    b.d_n_face_ids = scal.data_ptr()
    b.d_map = fmap.data_ptr()
    b.d_n_map = scal.data_ptr() + 4
    uf = cfg.use_filter if use_filter is None else use_filter
    wsb = lib.vf_bins_workspace_size(C.byref(c), F, int(level))
    ws = _ws.get("bins", wsb)
    _lib.check(lib.vf_build_bins(C.byref(c), _lib.ptr(dm.faces), F, int(level), _mode(mode),
                                 int(bool(uf)), C.byref(b), C.c_void_p(scal.data_ptr() + 8),
                                 _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "build_bin_hierarchy")
    h = scal.cpu().numpy()
    if h[2]:
        _lib.check(int(h[2]), "build_bin_hierarchy")
    P, K = int(h[0]), int(h[1])
    return BinLevel(level, cfg.bins(level), face_ids[:P], counts, offsets,
                    FilterMap(None, fmap[:K]), _mode(mode))


def build_bin_hierarchy(mesh, cfg: EmbedConfig = EmbedConfig(), mode=AXIS_ONLY,
                        l_max_b: Optional[int] = None) -> List[BinLevel]:
    """One BinLevel per level 0 <= L < L_max,B."""
    n = cfg.l_max if l_max_b is None else int(l_max_b)
    return [build_level(mesh, L, cfg, mode) for L in range(n)]
