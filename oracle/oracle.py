"""ctypes front-end of the CPU oracle (oracle/vf_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
bench's cpu_baseline / --impl reference leg, always as the checker or the CPU
baseline, never as the measured or shipped path.  See vf_oracle.h for the
reference citations and the parity status ("SAT pinned to reference golden
vectors; pipeline pinned to SPEC examples + independent oracles").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libvf_oracle.so")
MAX_LEVELS = 16

FLUID, SOLID, GUARD, GHOST, INTERFACE, BOUNDARY = range(6)
BF_SOLID, BF_SB, BF_SA, BF_MARK, BF_REFINED, BF_BOUNDARY = 1, 2, 4, 8, 16, 32


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "vf_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    return _LIB_PATH


class OrcConfig(C.Structure):
    _fields_ = [("nb", C.c_int32 * 3), ("l_max", C.c_int32), ("n_spec", C.c_int32),
                ("n_prop", C.c_int32), ("dx0", C.c_double), ("len", C.c_double * 3),
                ("eps_slab", C.c_double), ("eps_parallel", C.c_double)]


class OrcGrid(C.Structure):
    _fields_ = [("coords", C.c_void_p), ("nbr", C.c_void_p), ("nbr_child", C.c_void_p),
                ("child", C.c_void_p), ("bflags", C.c_void_p), ("masks", C.c_void_p),
                ("level_start", C.c_int32 * (MAX_LEVELS + 1)), ("n_levels", C.c_int32),
                ("capacity", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        i64, i32 = C.c_int64, C.c_int
        sig = {
            "orc_abi_version": (i32, []),
            "orc_set_threads": (None, [i32]),
            "orc_get_threads": (i32, []),
            "orc_sat_batch": (None, [P, P, i64, P]),
            "orc_ray_indicators": (i32, [P, P, i64, P, i32, i32, P]),
            "orc_compact": (i64, [P, i64, P]),
            "orc_bin_pairs": (i32, [P, i64, P, i64, P, i32, P, P, i64, P]),
            "orc_assemble": (None, [P, P, i64, i64, P, P, P]),
            "orc_init_forest": (i32, [P, P]),
            "orc_voxelize_level": (i32, [P, P, i32, P, P, P, P, P]),
            "orc_propagate": (i32, [P, P, i32, i32]),
            "orc_finalize": (i32, [P, P, i32]),
            "orc_mark": (i32, [P, P, i32]),
            "orc_adapt": (i32, [P, P, i32]),
            "orc_boundary": (i32, [P, P, P]),
            "orc_tables": (i64, [P, P, P]),
            "orc_link_lengths": (i32, [P, P, P, i64, P, P, P, P, P, P]),
            "orc_embed": (i32, [P, P, P, P, i64, i32, C.POINTER(P), P]),
            "orc_links_nb": (i64, [P]),
            "orc_op_counters": (None, [P]),
            "orc_links_copy": (None, [P, P, P]),
            "orc_links_free": (None, [P]),
            "orc_parity_inside": (None, [P, i64, P, i64, C.c_double, P]),
            "orc_lbm_equilibrium": (None, [C.c_double, P, P]),
            "orc_lbm_step": (i32, [P, P, P, i32, i32, i32, P, P, P, P, C.c_double, P, i32, i32, P]),
            "orc_lbm_fill_ghosts": (i32, [P, P, P, P, i32, i32, i32, i32, P, P, C.c_double, C.c_double,
                                          i32, P]),
            "orc_lbm_restrict": (i32, [P, P, i32, i32, i32, i32, P, C.c_double, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def make_config(cfg) -> OrcConfig:
    """From an EmbedConfig-like object (nb, l_max, n_spec, n_prop, dx0,
    domain, eps, eps_parallel)."""
    c = OrcConfig()
    c.nb[:] = list(cfg.nb)
    c.l_max = cfg.l_max
    c.n_spec = cfg.n_spec
    c.n_prop = cfg.n_prop
    c.dx0 = cfg.dx0
    c.len[:] = [float(x) for x in cfg.domain]
    c.eps_slab = cfg.eps
    c.eps_parallel = cfg.eps_parallel
    return c


def set_threads(n: int):
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return lib().orc_get_threads()


def _f64(a, cols):
    return np.ascontiguousarray(a, dtype=np.float64).reshape(-1, cols)


def sat_batch(tri, box):
    tri = _f64(tri, 9)
    box = _f64(box, 6)
    out = np.zeros(len(tri), dtype=np.uint8)
    lib().orc_sat_batch(_p(tri), _p(box), len(tri), _p(out))
    return out.astype(bool)


def ray_indicators(fc, nrm, cfg, L, mode=0):
    fc, nrm = _f64(fc, 9), _f64(nrm, 3)
    out = np.zeros(len(fc), dtype=np.uint8)
    c = make_config(cfg)
    rc = lib().orc_ray_indicators(_p(fc), _p(nrm), len(fc), C.byref(c), L, mode, _p(out))
    assert rc == 0
    return out


def compact(ind):
    ind = np.ascontiguousarray(ind, dtype=np.uint8)
    m = np.zeros(len(ind) + 1, dtype=np.int32)
    n = lib().orc_compact(_p(ind), len(ind), _p(m))
    return m[:n].copy()


def bin_pairs(fc, fmap, cfg, L):
    fc = _f64(fc, 9)
    fmap = np.ascontiguousarray(fmap, dtype=np.int32)
    cap = len(fmap) * cfg.n_lim + 1
    pb = np.zeros(cap, dtype=np.int32)
    pf = np.zeros(cap, dtype=np.int32)
    n = C.c_int64(0)
    c = make_config(cfg)
    rc = lib().orc_bin_pairs(_p(fc), len(fc), _p(fmap), len(fmap), C.byref(c), L,
                             _p(pb), _p(pf), cap, C.byref(n))
    if rc == 3:
        raise RuntimeError("N_lim pair cap violated (internal error, SPEC.md:146)")
    assert rc == 0, rc
    return pb[:n.value].copy(), pf[:n.value].copy()


def assemble(pb, pf, n_bins):
    pb = np.ascontiguousarray(pb, dtype=np.int32)
    pf = np.ascontiguousarray(pf, dtype=np.int32)
    counts = np.zeros(n_bins, dtype=np.int32)
    offsets = np.zeros(n_bins, dtype=np.int32)
    face_ids = np.zeros(len(pb) + 1, dtype=np.int32)
    lib().orc_assemble(_p(pb), _p(pf), len(pb), n_bins, _p(counts), _p(offsets), _p(face_ids))
    return counts, offsets, face_ids[:len(pb)].copy()


def build_bins(fc, nrm, cfg, L, mode=0, use_filter=True):
    if use_filter:
        fmap = compact(ray_indicators(fc, nrm, cfg, L, mode))
    else:
        fmap = np.arange(len(fc), dtype=np.int32)
    pb, pf = bin_pairs(fc, fmap, cfg, L)
    return assemble(pb, pf, cfg.n_bins(L))


@dataclass
class Grid:
    """numpy-owned forest arrays in the layout shared with the GPU path."""
    coords: np.ndarray      # (cap, 4) int32: i, j, k, level
    nbr: np.ndarray         # (cap, 27) int32
    nbr_child: np.ndarray   # (cap, 27) int32
    child: np.ndarray       # (cap,) int32
    bflags: np.ndarray      # (cap,) uint8
    masks: np.ndarray       # (cap, 64) uint8
    level_start: np.ndarray  # (17,) int32
    n_levels: int

    @classmethod
    def empty(cls, capacity):
        return cls(np.zeros((capacity, 4), np.int32), np.zeros((capacity, 27), np.int32),
                   np.zeros((capacity, 27), np.int32), np.zeros(capacity, np.int32),
                   np.zeros(capacity, np.uint8), np.zeros((capacity, 64), np.uint8),
                   np.zeros(MAX_LEVELS + 1, np.int32), 0)

    @property
    def capacity(self):
        return len(self.child)

    @property
    def n_used(self):
        return int(self.level_start[self.n_levels])

    def level_range(self, L):
        return int(self.level_start[L]), int(self.level_start[L + 1])

    def copy(self):
        return Grid(self.coords.copy(), self.nbr.copy(), self.nbr_child.copy(), self.child.copy(),
                    self.bflags.copy(), self.masks.copy(), self.level_start.copy(), self.n_levels)

    def _struct(self):
        g = OrcGrid()
        g.coords, g.nbr, g.nbr_child = _p(self.coords), _p(self.nbr), _p(self.nbr_child)
        g.child, g.bflags, g.masks = _p(self.child), _p(self.bflags), _p(self.masks)
        g.level_start[:] = [int(x) for x in self.level_start]
        g.n_levels = self.n_levels
        g.capacity = self.capacity
        return g

    def _sync(self, g):
        self.level_start[:] = list(g.level_start)
        self.n_levels = int(g.n_levels)

    def call(self, name, cfg, *args):
        g = self._struct()
        c = make_config(cfg)
        rc = getattr(lib(), name)(C.byref(g), C.byref(c), *args)
        self._sync(g)
        return rc


def init_forest(cfg, capacity):
    g = Grid.empty(capacity)
    rc = g.call("orc_init_forest", cfg)
    if rc:
        raise RuntimeError(f"init_forest rc={rc}")
    return g


def voxelize_level(g, cfg, L, bins, fc, nrm):
    counts, offsets, face_ids = (np.ascontiguousarray(a, dtype=np.int32) for a in bins)
    fc, nrm = _f64(fc, 9), _f64(nrm, 3)
    assert g.call("orc_voxelize_level", cfg, L, _p(counts), _p(offsets), _p(face_ids),
                  _p(fc), _p(nrm)) == 0


def propagate(g, cfg, L, direction):
    assert g.call("orc_propagate", cfg, L, int(direction)) == 0


def finalize(g, cfg, L):
    assert g.call("orc_finalize", cfg, L) == 0


def mark(g, cfg, L):
    assert g.call("orc_mark", cfg, L) == 0


def adapt(g, cfg, L):
    rc = g.call("orc_adapt", cfg, L)
    if rc == 2:
        raise MemoryError("forest capacity exhausted at level %d" % L)
    assert rc == 0, rc


def boundary(g, cfg):
    bcount = np.zeros(g.capacity, dtype=np.int32)
    assert g.call("orc_boundary", cfg, _p(bcount)) == 0
    return bcount


def tables(g, bcount):
    cmap = np.zeros(max(g.n_used, 1), dtype=np.int32)
    gs = g._struct()
    nb = lib().orc_tables(C.byref(gs), _p(np.ascontiguousarray(bcount, np.int32)), _p(cmap))
    return int(nb), cmap[:g.n_used].copy()


def link_lengths(g, cfg, cmap, n_b, md_bins, fc, nrm):
    counts, offsets, face_ids = (np.ascontiguousarray(a, dtype=np.int32) for a in md_bins)
    fc, nrm = _f64(fc, 9), _f64(nrm, 3)
    lengths = np.zeros(max(n_b, 1) * 27 * 64, dtype=np.float32)
    cmap = np.ascontiguousarray(cmap, dtype=np.int32)
    gs = g._struct()
    c = make_config(cfg)
    rc = lib().orc_link_lengths(C.byref(gs), C.byref(c), _p(cmap), n_b, _p(counts), _p(offsets),
                                _p(face_ids), _p(fc), _p(nrm), _p(lengths))
    assert rc == 0
    return lengths[:n_b * 27 * 64].reshape(n_b, 27, 64)


@dataclass
class EmbedResult:
    grid: Grid
    n_b: int
    contraction_map: np.ndarray
    lengths: np.ndarray           # (n_b, 27, 64) float32
    stage_seconds: np.ndarray     # see orc_embed


def embed(fc, nrm, cfg, capacity, use_filter=True):
    fc, nrm = _f64(fc, 9), _f64(nrm, 3)
    g = Grid.empty(capacity)
    gs = g._struct()
    c = make_config(cfg)
    h = C.c_void_p()
    st = np.zeros(8, dtype=np.float64)
    rc = lib().orc_embed(C.byref(gs), C.byref(c), _p(fc), _p(nrm), len(fc), int(use_filter),
                         C.byref(h), _p(st))
    g._sync(gs)
    if rc == 2:
        raise MemoryError("forest capacity exhausted")
    if rc:
        raise RuntimeError(f"orc_embed rc={rc}")
    nb = int(lib().orc_links_nb(h))
    cmap = np.zeros(max(g.n_used, 1), dtype=np.int32)
    lengths = np.zeros(max(nb, 1) * 27 * 64, dtype=np.float32)
    lib().orc_links_copy(h, _p(cmap), _p(lengths))
    lib().orc_links_free(h)
    return EmbedResult(g, nb, cmap[:g.n_used].copy(), lengths[:nb * 27 * 64].reshape(nb, 27, 64), st)


OP_STAGES = ("indicators", "pairs", "voxelize", "md_bins", "link_lengths")


def op_counters():
    """Algorithmic operation counts of the last embed() (then reset), per
    stage: {stage: {"sat_calls", "sat_ops", "other_ops"}}."""
    out = np.zeros((5, 3), dtype=np.uint64)
    lib().orc_op_counters(_p(out))
    return {k: {"sat_calls": int(r[0]), "sat_ops": int(r[1]), "other_ops": int(r[2])}
            for k, r in zip(OP_STAGES, out)}


def parity_inside(fc, pts, tol=1e-9):
    fc = _f64(fc, 9)
    pts = _f64(pts, 3)
    out = np.zeros(len(pts), dtype=np.uint8)
    lib().orc_parity_inside(_p(fc), len(fc), _p(pts), len(pts), float(tol), _p(out))
    return out


# ---------------------------------------------------------------------------
# LUT consumer (lbm_oracle.c): D3Q27 BGK collide/stream of one level


def lbm_equilibrium(rho, u):
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros(27)
    lib().orc_lbm_equilibrium(float(rho), _p(u), _p(out))
    return out


def lbm_step(coords, nbr, masks, s, e, cells_x, cmap, lengths, fin, tau, u_in, ibb=True,
             open_x=True):
    """One step of level blocks [s, e); fin = (27, (e-s)*64)
    float32 post-collision populations.  Returns (fout, force[3])."""
    coords = np.ascontiguousarray(coords, dtype=np.int32)
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    masks = np.ascontiguousarray(masks, dtype=np.uint8)
    cmap = np.ascontiguousarray(cmap, dtype=np.int32)
    lengths = np.ascontiguousarray(lengths, dtype=np.float32)
    fin = np.ascontiguousarray(fin, dtype=np.float32)
    fout = np.zeros_like(fin)
    u = np.ascontiguousarray(u_in, dtype=np.float64)
    force = np.zeros(3)
    rc = lib().orc_lbm_step(_p(coords), _p(nbr), _p(masks), int(s), int(e), int(cells_x), _p(cmap),
                            _p(lengths), _p(fin), _p(fout), float(tau), _p(u), int(bool(ibb)),
                            int(bool(open_x)), _p(force))
    assert rc == 0
    return fout, force


# interface exchange + step_hierarchy (lbm_oracle.c)


def lbm_fill_ghosts(g, sf, ef, sc, ec, fc_old, fc_new, theta, alpha, order, ff):
    """Fine GHOST cells of blocks [sf, ef) from the coarse level [sc, ec);
    returns a new fine state (27, (ef-sf)*64)."""
    out = np.ascontiguousarray(ff, dtype=np.float32).copy()
    fo = np.ascontiguousarray(fc_old, dtype=np.float32)
    fn = np.ascontiguousarray(fc_new if fc_new is not None else fc_old, dtype=np.float32)
    rc = lib().orc_lbm_fill_ghosts(_p(np.ascontiguousarray(g["coords"], dtype=np.int32)),
                                   _p(np.ascontiguousarray(g["nbr"], dtype=np.int32)),
                                   _p(np.ascontiguousarray(g["masks"], dtype=np.uint8)),
                                   _p(np.ascontiguousarray(g["child"], dtype=np.int32)), int(sf), int(ef),
                                   int(sc), int(ec), _p(fo), _p(fn), float(theta), float(alpha), int(order),
                                   _p(out))
    assert rc == 0
    return out


def lbm_restrict(g, sc, ec, sf, ef, ff, beta, fc):
    """Coarse cells of refined blocks in [sc, ec) from their children in
    [sf, ef); returns a new coarse state."""
    out = np.ascontiguousarray(fc, dtype=np.float32).copy()
    rc = lib().orc_lbm_restrict(_p(np.ascontiguousarray(g["masks"], dtype=np.uint8)),
                                _p(np.ascontiguousarray(g["child"], dtype=np.int32)), int(sc), int(ec), int(sf),
                                int(ef), _p(np.ascontiguousarray(ff, dtype=np.float32)), float(beta), _p(out))
    assert rc == 0
    return out


def level_taus(tau0, n_levels):
    """Acoustic scaling: nu_L = 2^L nu_0, tau_L = 3 nu_L + 1/2."""
    nu0 = (tau0 - 0.5) / 3.0
    return [3.0 * nu0 * 2 ** L + 0.5 for L in range(n_levels)]


def neq_factors(tau_c, tau_f):
    """Post-collision non-equilibrium rescale coarse -> fine (alpha) and
    fine -> coarse (beta = 1 / alpha): (tau_f - 1) / (2 (tau_c - 1))."""
    if abs(tau_c - 1.0) < 1e-9 or abs(tau_f - 1.0) < 1e-9:
        raise ValueError("tau_L = 1 loses the non-equilibrium part of post-collision populations")
    a = (tau_f - 1.0) / (2.0 * (tau_c - 1.0))
    return a, 1.0 / a


def lbm_step_hierarchy(g, ranges, cells_x0, cmap, lengths, states, tau0, u_in, ibb=True, open_x=True,
                       order=3, rescale=True):
    """One coarse step of the level hierarchy: level L
    advances, then level L+1 takes two substeps with its ghosts filled from L
    at theta = 0 and 1/2, then L's covered cells are restricted from L+1.
    ranges[L] = (s, e); states[L] = (27, (e-s)*64) float32.  Returns the new
    states and the number of collide/stream steps per level."""
    n = len(ranges)
    taus = level_taus(tau0, n)
    states = [np.array(x, dtype=np.float32, copy=True) for x in states]
    counts = [0] * n

    def advance(L):
        s, e = ranges[L]
        old = states[L]
        states[L], _ = lbm_step(g["coords"], g["nbr"], g["masks"], s, e, cells_x0 << L, cmap, lengths, old,
                                taus[L], u_in, ibb, open_x)
        counts[L] += 1
        if L + 1 < n:
            sf, ef = ranges[L + 1]
            a, b = neq_factors(taus[L], taus[L + 1]) if rescale else (1.0, 1.0)
            for th in (0.0, 0.5):
                states[L + 1] = lbm_fill_ghosts(g, sf, ef, s, e, old, states[L], th, a, order, states[L + 1])
                advance(L + 1)
            states[L] = lbm_restrict(g, s, e, sf, ef, states[L + 1], b, states[L])

    advance(0)
    return states, counts
