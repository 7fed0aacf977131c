"""ctypes binding of libvoxforest_b200.so (include/voxforest_b200.h).

The shared library is built in-tree (``__graft_entry__.build()`` or
``make -C paper_2512_01251_b200/csrc``).  There is no CPU fallback: if the
library is missing or no CUDA device is present, every GPU op raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import (BinCapError, CapacityError, CudaError, MeshError, VoxforestError)

_HERE = os.path.dirname(os.path.abspath(__file__))
# VF_LIB_PATH: an alternative in-tree build of the same library (A/B kernel experiments)
LIB_PATH = os.environ.get("VF_LIB_PATH") or os.path.join(_HERE, "libvoxforest_b200.so")
ABI_VERSION = 6
MAX_LEVELS = 16

# cell masks / block flags / neighbour codes (voxforest_b200.h)
FLUID, SOLID, GUARD, GHOST, INTERFACE, BOUNDARY = range(6)
BF_SOLID, BF_SB, BF_SA, BF_MARK, BF_REFINED, BF_BOUNDARY = 1, 2, 4, 8, 16, 32
NB_OUTSIDE, NB_MISSING, NB_SOLID_NBR = -1, -2, -3


class VfConfig(C.Structure):
    _fields_ = [("nb", C.c_int32 * 3), ("l_max", C.c_int32), ("n_spec", C.c_int32),
                ("n_prop", C.c_int32), ("dx0", C.c_double), ("len", C.c_double * 3),
                ("eps_slab", C.c_double), ("eps_parallel", C.c_double),
                ("shard_rank", C.c_int32), ("shard_count", C.c_int32),
                ("d_row_owner", C.c_void_p), ("pair_cap", C.c_int64),
                ("line_cap", C.c_int64)]


class VfGrid(C.Structure):
    _fields_ = [("d_coords", C.c_void_p), ("d_nbr", C.c_void_p), ("d_nbr_child", C.c_void_p),
                ("d_child", C.c_void_p), ("d_bflags", C.c_void_p), ("d_masks", C.c_void_p),
                ("d_level_start", C.c_void_p), ("d_status", C.c_void_p),
                ("d_solid64", C.c_void_p), ("capacity", C.c_int32), ("n_levels", C.c_int32)]


class VfBins(C.Structure):
    _fields_ = [("level", C.c_int32), ("mode", C.c_int32), ("d_counts", C.c_void_p),
                ("d_offsets", C.c_void_p), ("d_face_ids", C.c_void_p),
                ("face_ids_cap", C.c_int64), ("d_n_face_ids", C.c_void_p),
                ("d_map", C.c_void_p), ("d_n_map", C.c_void_p)]


_P, _I64, _I32, _SZ = C.c_void_p, C.c_int64, C.c_int, C.c_size_t
_CP = C.POINTER(VfConfig)
_GP = C.POINTER(VfGrid)
_BP = C.POINTER(VfBins)

_SIGS = {
    "vf_abi_version": (_I32, []),
    "vf_ctx_create": (_P, [_I32, _P]),
    "vf_ctx_destroy": (_I32, [_P]),
    "vf_ctx_device": (_I32, [_P]),
    "vf_nccl_unique_id": (_I32, [_P, _I32]),
    "vf_ctx_create_nccl": (_P, [_I32, _I32, _I32, _P]),
    "vf_shard_embed_phase1": (_I32, [_P, _CP, _P, _I64, _I32, _GP, _P, _P, _P, _P, _SZ, _P]),
    "vf_last_error": (C.c_char_p, []),
    "vf_device_info": (_I32, [C.POINTER(C.c_int)] * 3),
    "vf_pack_faces": (_I32, [_P, _P, _I64, _P, _P]),
    "vf_sat_batch": (_I32, [_P, _P, _I64, _P, _P]),
    "vf_bins_workspace_size": (_SZ, [_CP, _I64, _I32]),
    "vf_ray_indicators": (_I32, [_CP, _P, _I64, _I32, _I32, _P, _P]),
    "vf_compact_workspace_size": (_SZ, [_I64]),
    "vf_assemble_workspace_size": (_SZ, [_I64, _I64]),
    "vf_compact": (_I32, [_P, _I64, _P, _P, _P, _SZ, _P]),
    "vf_bin_pairs": (_I32, [_CP, _P, _I64, _P, _P, _I32, _P, _P, _I64, _P, _P, _P, _SZ, _P]),
    "vf_bin_assemble": (_I32, [_P, _P, _P, _I64, _I64, _P, _P, _P, _P, _SZ, _P]),
    "vf_build_bins": (_I32, [_CP, _P, _I64, _I32, _I32, _I32, _BP, _P, _P, _SZ, _P]),
    "vf_init_forest": (_I32, [_CP, _GP, _P]),
    "vf_adapt_workspace_size": (_SZ, [_GP]),
    "vf_adapt_refine": (_I32, [_CP, _GP, _I32, _P, _SZ, _P]),
    "vf_voxelize_level": (_I32, [_CP, _GP, _I32, _BP, _P, _P]),
    "vf_propagate_workspace_size": (_SZ, [_GP]),
    "vf_propagate_x": (_I32, [_CP, _GP, _I32, _I32, _I32, _P, _SZ, _P]),
    "vf_finalize_level": (_I32, [_CP, _GP, _I32, _P]),
    "vf_mark_workspace_size": (_SZ, [_GP]),
    "vf_mark_level": (_I32, [_CP, _GP, _I32, _P, _SZ, _P]),
    "vf_boundary_cells": (_I32, [_CP, _GP, _P, _P]),
    "vf_tables_workspace_size": (_SZ, [_GP]),
    "vf_link_tables": (_I32, [_CP, _GP, _P, _P, _P, _P, _SZ, _P]),
    "vf_link_workspace_size": (_SZ, [_CP, _GP]),
    "vf_link_lengths": (_I32, [_CP, _GP, _P, _P, _I64, _P, _P, _P, _P, _SZ, _P]),
    "vf_embed_workspace_size": (_SZ, [_CP, _I64, C.c_int32]),
    "vf_embed_phase1": (_I32, [_CP, _P, _I64, _I32, _GP, _P, _P, _P, _SZ, _P, C.POINTER(_P)]),
    "vf_embed_phase2": (_I32, [_CP, _P, _I64, _GP, _P, _P, _P, _I64, _P, _SZ, _P, C.POINTER(_P)]),
    "vf_embed_graph_create": (_I32, [_CP, _P, _I64, _I32, _GP, _P, _P, _P, _I64, _P, _SZ, _P,
                                     C.POINTER(_P)]),
    "vf_graph_launch": (_I32, [_P, _P]),
    "vf_graph_destroy": (None, [_P]),
    "vf_launch_count": (_I64, []),
    "vf_ktimer_start": (_I32, [_P, C.c_double]),
    "vf_pack_indexed": (_I32, [_P, _I64, _P, _I64, _P, _P, _P]),
    "vf_lut_sparse_workspace_size": (_SZ, [_I64]),
    "vf_lut_sparse": (_I32, [_P, _I64, _P, _P, _P, _I64, _P, _P, _SZ, _P]),
    "vf_ktimer_stop": (_I32, [C.c_char_p, _I32]),
    "vf_embed_link_stats": (_I32, [_CP, _I64, _I32, _P, _SZ, _P]),
    "vf_side_sync": (_I32, []),
    "vf_check_status": (_I32, [_GP, _P]),
    "vf_shard_zero_unowned": (_I32, [_CP, _GP, _I32, _P, _P]),
    "vf_set_link_band_cap": (_I64, [_I64]),
    "vf_set_serial_links": (_I32, [_I32]),
    "vf_set_link_small_ext": (C.c_float, [C.c_float]),
    "vf_shard_owner_bytes": (_SZ, [_CP]),
    "vf_shard_owner_map": (_I32, [_CP, _GP, _I32, _P, _SZ, _P]),
    "vf_shard_level": (_I32, [_CP, _P, _I64, _I32, _GP, _I32, _P, _SZ, _P]),
    "vf_shard_refine": (_I32, [_CP, _GP, _I32, _P, _SZ, _P]),
    "vf_shard_boundary": (_I32, [_CP, _GP, _P, _P]),
    "vf_shard_links": (_I32, [_CP, _P, _I64, _GP, _P, _P, _P, _I64, _P, _SZ, _P]),
    "vf_lbm_init": (_I32, [_GP, C.c_int32, C.c_int32, C.c_double, _P, _P, _P]),
    "vf_stl_workspace_size": (_SZ, [_I64]),
    "vf_stl_scan": (_I32, [_P, _I64, _P, _SZ, _P, _P, _P, _P]),
    "vf_stl_weld_workspace_size": (_SZ, [_I64]),
    "vf_stl_build": (_I32, [_P, _I64, _P, _SZ, _I64, C.c_double, _P, _SZ, _P, _P, _P, _P, _P, _P, _P, _P]),
    "vf_lbm_step": (_I32, [_CP, _GP, _I32, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "vf_lbm_parents": (_I32, [_GP, C.c_int32, _P, _P]),
    "vf_lbm_fill_ghosts": (_I32, [_GP, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, C.c_double,
                                  C.c_double, _I32, _P, _P]),
    "vf_lbm_restrict": (_I32, [_GP, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, _P, C.c_double, _P, _P]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load and type the shared library (no CUDA context needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise VoxforestError(
                f"CUDA extension not built ({path} missing): run __graft_entry__.build() "
                "or `make -C paper_2512_01251_b200/csrc`; there is no CPU fallback")
        lib = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        if lib.vf_abi_version() != ABI_VERSION:
            raise VoxforestError("libvoxforest_b200 ABI mismatch")
        _lib = lib
        return lib


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise CudaError("no CUDA device: the B200 engine has no CPU fallback")
    return load()


def last_error() -> str:
    return (load().vf_last_error() or b"").decode()


def check(rc: int, what: str = ""):
    if rc == 0:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise CapacityError(msg)
    if rc == 3:
        raise BinCapError(msg)
    if rc == 4:
        raise CudaError(msg)
    if rc == 6:
        raise MeshError(msg)
    raise VoxforestError(f"rc={rc}: {msg}")


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def make_config(cfg, shard=(0, 1)) -> VfConfig:
    """vf_config from an EmbedConfig; ``shard`` = (rank, n_ranks) for the
    block-sharded multi-GPU embed (row ownership, see include/voxforest_b200.h)."""
    c = VfConfig()
    c.shard_rank, c.shard_count = int(shard[0]), int(shard[1])
    c.nb[:] = list(cfg.nb)
    c.l_max = cfg.l_max
    c.n_spec = cfg.n_spec
    c.n_prop = cfg.n_prop
    c.dx0 = cfg.dx0
    c.len[:] = [float(x) for x in cfg.domain]
    c.eps_slab = cfg.eps
    c.eps_parallel = cfg.eps_parallel
    return c


__all__ = ["load", "require_cuda", "check", "make_config", "VfConfig", "VfGrid", "VfBins",
           "stream_ptr", "ptr", "EXPORTED", "MeshError"]
