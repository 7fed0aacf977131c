"""CPU suite: pins the oracle (test infrastructure) against the reference's
golden vectors, the SPEC worked examples and independent oracles.  No GPU."""
import os

import numpy as np
import pytest

from paper_2512_01251_b200 import EmbedConfig, make_icosphere, make_torus
from paper_2512_01251_b200.lattice import D3Q27_C, D3Q27_OPPOSITE
from paper_2512_01251_b200.mesh import TriangleMesh, l_spec_bound, refine_faces, translate

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def O(oracle_mod):
    return oracle_mod


# ---------------------------------------------------------------- pins
def test_sat_matches_reference_golden(O):
    z = np.load(os.path.join(GOLD, "sat_golden.npz"))
    got = O.sat_batch(z["tri"], z["box"])
    assert np.array_equal(got, z["out"]), int((got != z["out"]).sum())
    assert 0 < z["out"].sum() < len(z["out"])


def test_lattice_matches_reference_golden():
    z = np.load(os.path.join(GOLD, "lattice_golden.npz"))
    assert np.array_equal(D3Q27_C, z["c"])
    assert np.array_equal(D3Q27_OPPOSITE, z["opposite"])


def test_icosphere_matches_reference_golden():
    z = np.load(os.path.join(GOLD, "mesh_golden.npz"))
    m = make_icosphere((0.5, 0.5, 0.5), 0.5, 2)
    assert np.array_equal(m.faces_indexed, z["faces"])
    # numpy's 1-D norm goes through host BLAS in the reference: <= 1 ulp apart
    assert np.abs(m.vertices - z["vertices"]).max() <= 2.3e-16
    assert np.abs(m.normals - z["normals"]).max() <= 1e-14


REF = "/root/reference/pkg/src/voxforest"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted (GPU box)")
def test_sat_matches_live_reference(O, tmp_path, monkeypatch):
    monkeypatch.setenv("NUMBA_CACHE_DIR", str(tmp_path))
    import importlib.util
    import sys
    spec = importlib.util.spec_from_file_location("vref_geometry_t", os.path.join(REF, "geometry.py"))
    g = importlib.util.module_from_spec(spec)
    sys.modules["vref_geometry_t"] = g
    spec.loader.exec_module(g)
    rng = np.random.default_rng(7)
    tri = rng.integers(0, 16, size=(3000, 9)) / 16.0
    lo = rng.integers(0, 16, size=(3000, 3)) / 16.0
    box = np.concatenate([lo, lo + rng.integers(0, 5, size=(3000, 3)) / 16.0], axis=1)
    ref = np.array([g.tri_aabb_overlap_3d(*t, *b) for t, b in zip(tri, box)])
    assert np.array_equal(O.sat_batch(tri, box), ref)
    # ray_face_distance: reference uses numpy/BLAS dots (geometry.py:434-437);
    # the pinned association (A7) agrees to a few ulp
    for _ in range(200):
        v = rng.random((3, 3))
        o = rng.random(3)
        n = np.cross(v[1] - v[0], v[2] - v[0])
        n = n / np.linalg.norm(n)
        r = g.ray_face_distance(o, np.array([1.0, 0, 0]), v, n)
        if r is None:
            continue
        num = (v[0, 0] - o[0]) * n[0] + ((v[0, 1] - o[1]) * n[1] + (v[0, 2] - o[2]) * n[2])
        d = num / n[0]
        assert abs(d - r[0]) <= 8 * np.spacing(max(abs(d), 1e-300)) + 1e-15


# ---------------------------------------------------------------- SPEC examples
def test_compaction_example(O):
    assert O.compact(np.array([0, 1, 1, 0, 1], np.uint8)).tolist() == [1, 2, 4]
    assert O.compact(np.zeros(7, np.uint8)).tolist() == []


def test_assemble_example(O):
    c, o, f = O.assemble(np.array([2, 0, 2], np.int32), np.array([0, 1, 3], np.int32), 4)
    assert c.tolist() == [1, 0, 2, 0] and o[0] == 0 and o[2] == 1 and f.tolist() == [1, 0, 3]


def test_l_spec_example():
    assert abs(l_spec_bound((1.0, 1.0, 1.0), 2, 5, 16) - 1.9 / 256) < 1e-15


def test_n_prop_example():
    assert EmbedConfig(n_x=512, d_spec=0.05).n_prop == 5
    assert EmbedConfig(n_x=64, d_spec=0.05).n_prop == 1
    assert EmbedConfig(n_x=64, d_spec=0.0).n_prop == 1


def test_index_maps_examples():
    from paper_2512_01251_b200.forest import index_maps
    assert index_maps((1, 2, 3), (0, 0, 0))[0] == 57
    t, th, Ip, v = index_maps((3, 1, 2), (1, 0, 0))
    assert Ip == (0, 1, 2) and v
    t, th, Ip, v = index_maps((1, 1, 1), (1, 0, 0))
    assert Ip == (2, 1, 1) and not v


def test_index_maps_spec_formula_and_neighbor_direction():
    """Every (I, c): the SPEC.md:229 violation flag literally (AND over the
    axes), and the general neighbour-block direction of pin A15 the kernels
    use: cell I + c lies in the block at neighbor_direction(I, c), at I'."""
    import itertools
    from paper_2512_01251_b200.forest import index_maps, neighbor_direction
    from paper_2512_01251_b200.lattice import D3Q27_C
    for I in itertools.product(range(4), repeat=3):
        for c in D3Q27_C:
            t, th, Ip, v = index_maps(I, c)
            assert t == I[0] + 4 * I[1] + 16 * I[2] and th == (I[0] + 1) + 6 * (I[1] + 1) + 36 * (I[2] + 1)
            assert v == all((Ip[d] != I[d] + c[d]) or c[d] == 0 for d in range(3))
            nd = neighbor_direction(I, c)
            for d in range(3):
                assert 4 * nd[d] + Ip[d] == I[d] + c[d]


def test_init_forest_links(O):
    cfg = EmbedConfig(n_x=16, l_max=2)
    g = O.init_forest(cfg, 64)
    assert g.n_used == 64
    # corner block 0: every slot with a negative component is outside
    for q, c in enumerate(D3Q27_C):
        if q and np.any(c < 0):
            assert g.nbr[0, q] == -1
    # involutive links
    for b in range(64):
        for q in range(1, 27):
            n = g.nbr[b, q]
            if n >= 0:
                assert g.nbr[n, D3Q27_OPPOSITE[q]] == b


def test_bin_pairs_examples(O):
    cfg = EmbedConfig(n_x=16, l_max=1)  # 4^3 bins of 0.25, dx = 1/16
    tiny = np.array([[0.60, 0.60, 0.60, 0.61, 0.60, 0.60, 0.60, 0.61, 0.60]])
    pb, pf = O.bin_pairs(tiny, np.array([0], np.int32), cfg, 0)
    assert len(pb) == 1 and pb[0] == 2 + 4 * (2 + 4 * 2)
    out = tiny + 2.0
    pb, _ = O.bin_pairs(out, np.array([0], np.int32), cfg, 0)
    assert len(pb) == 0


def test_bin_pairs_vs_exhaustive_scan(O):
    """pair multiset equals the all-bins x all-faces scan."""
    m = translate(make_torus(24, 12), (0.013, 0.007, -0.004))
    cfg = EmbedConfig(n_x=32, l_max=2)
    for L in (0, 1):
        pb, pf = O.bin_pairs(m.faces_coord, np.arange(m.n_faces, dtype=np.int32), cfg, L)
        B = cfg.bins(L)
        h, dx = 4 * cfg.dx(L), cfg.dx(L)
        want = set()
        ii = np.arange(B[0])
        for f in range(m.n_faces):
            tri = np.repeat(m.faces_coord[f:f + 1], B[0] ** 3, axis=0)
            I, J, K = np.meshgrid(ii, ii, ii, indexing="ij")
            I, J, K = I.ravel(), J.ravel(), K.ravel()
            box = np.stack([I * h - dx, J * h - dx, K * h - dx,
                            (I + 1) * h + dx, (J + 1) * h + dx, (K + 1) * h + dx], 1)
            hit = O.sat_batch(tri, box)
            for b in (I + B[0] * (J + B[1] * K))[hit]:
                want.add((int(b), f))
        assert set(zip(pb.tolist(), pf.tolist())) == want
        assert len(pb) == len(want)


def test_voxelize_sign_rule(O):
    """SPEC.md:289-290 on a box: centres just inside are solid, outside guard."""
    lo, hi = 0.3 + 1 / 128, 0.7 - 1 / 256
    v = np.array([[x, y, z] for z in (lo, hi) for y in (lo, hi) for x in (lo, hi)])
    quads = [[0, 2, 3, 1], [4, 5, 7, 6], [0, 1, 5, 4], [2, 6, 7, 3], [0, 4, 6, 2], [1, 3, 7, 5]]
    faces = [[q[0], q[1], q[2]] for q in quads] + [[q[0], q[2], q[3]] for q in quads]
    m = TriangleMesh(v, faces)
    cfg = EmbedConfig(n_x=32, l_max=1)
    g = O.init_forest(cfg, 512)
    bins = O.build_bins(m.faces_coord, m.normals, cfg, 0)
    O.voxelize_level(g, cfg, 0, bins, m.faces_coord, m.normals)
    O.propagate(g, cfg, 0, +1)
    O.finalize(g, cfg, 0)
    dx = cfg.dx(0)
    for b in range(512):
        co = g.coords[b, :3]
        for t in range(64):
            p = (4 * co + np.array([t & 3, (t >> 2) & 3, t >> 4]) + 0.5) * dx
            inside = np.all(p > lo) and np.all(p < hi)
            assert (g.masks[b, t] == 1) == inside


# ---------------------------------------------------------------- independent oracles
def _centers(g, cfg, L):
    s, e = g.level_range(L)
    co = g.coords[s:e, :3].astype(np.int64)
    t = np.arange(64)
    I = np.stack([t & 3, (t >> 2) & 3, t >> 4], 1)
    return ((4 * co[:, None, :] + I[None]) + 0.5) * cfg.dx(L)


@pytest.fixture(scope="module")
def c1(O):
    m = make_icosphere((0.5, 0.5, 0.5), 0.5, 4)
    cfg = EmbedConfig(n_x=32, l_max=3)
    r = O.embed(m.faces_coord, m.normals, cfg, cfg.block_capacity(m.face_areas().sum()))
    return m, cfg, r


def test_ray_parity_all_levels(O, c1):
    """SPEC.md:357 / acceptance #1: final solid masks equal the all-faces
    ray-parity oracle on every level away from eps of the surface."""
    m, cfg, r = c1
    g = r.grid
    for L in range(g.n_levels):
        P = _centers(g, cfg, L).reshape(-1, 3)
        par = O.parity_inside(m.faces_coord, P, 1e-9)
        s, e = g.level_range(L)
        sol = (g.masks[s:e].reshape(-1) == 1)
        ok = par != 2
        assert ok.mean() > 0.98
        assert np.array_equal(sol[ok], par[ok] == 1), L


def test_solid_volume(O, c1):
    """leaf solid volume within 1% of the analytic sphere."""
    m, cfg, r = c1
    g = r.grid
    vol = 0.0
    for L in range(g.n_levels):
        s, e = g.level_range(L)
        leaf = g.child[s:e] < 0
        vol += (g.masks[s:e][leaf] == 1).sum() * cfg.dx(L) ** 3
    assert abs(vol / (np.pi / 6 * 0.5 ** 3) - 1) < 0.01


def test_balance_and_topology(O, c1):
    """links involutive, children contiguous, 2:1 balance."""
    m, cfg, r = c1
    g = r.grid
    n = g.n_used
    lvl = g.coords[:n, 3]
    for b in range(n):
        for q in range(1, 27):
            v = g.nbr[b, q]
            if v >= 0:
                assert g.nbr[v, D3Q27_OPPOSITE[q]] == b
                assert lvl[v] == lvl[b]
        c = g.child[b]
        if c >= 0:
            assert np.all(g.coords[c:c + 8, 3] == lvl[b] + 1)
            assert np.all(g.coords[c:c + 8, :3] // 2 == g.coords[b, :3])
    # 2:1 balance: every leaf's missing same-level neighbour is covered by a
    # leaf exactly one level coarser (codes -2/-3 only refer to the parent's
    # existing unrefined neighbour)
    for b in range(n):
        if lvl[b] == 0:
            continue
        for q in range(1, 27):
            if g.nbr[b, q] in (-2, -3):
                pc = (g.coords[b, :3] + D3Q27_C[q]) // 2
                L = lvl[b] - 1
                s, e = g.level_range(L)
                hit = np.where(np.all(g.coords[s:e, :3] == pc, axis=1))[0]
                assert len(hit) == 1 and g.child[s + hit[0]] < 0


def test_marking_bfs(O):
    """marked set = BFS from the solid boundary."""
    m = translate(make_torus(60, 30), (0.004, 0.002, -0.003))
    cfg = EmbedConfig(n_x=32, l_max=2, d_spec=0.2)
    assert cfg.n_prop > 1
    g = O.init_forest(cfg, 20000)
    bins = O.build_bins(m.faces_coord, m.normals, cfg, 0)
    O.voxelize_level(g, cfg, 0, bins, m.faces_coord, m.normals)
    O.propagate(g, cfg, 0, +1)
    O.finalize(g, cfg, 0)
    O.mark(g, cfg, 0)
    s, e = g.level_range(0)
    solid = (g.bflags[s:e] & 1) > 0
    nb = g.nbr[s:e, 1:]
    ex = nb >= 0
    sb = solid & np.any(ex & ~solid[np.where(ex, nb, 0)], axis=1)
    # level 0 has no interface: every block eligible
    dist = np.full(e - s, 99)
    frontier = set(np.where(sb)[0])
    for b in frontier:
        dist[b] = 0
    d = 0
    while frontier:
        d += 1
        nxt = set()
        for b in frontier:
            for v in nb[b]:
                if v >= 0 and dist[v] == 99:
                    dist[v] = d
                    nxt.add(v)
        frontier = nxt
    # hop 1 from SB: everything; hop 2: solid too (first sweep); beyond: fluid only
    want = (dist <= 1)
    # sweeps: it=0 admits any block at hop 2; it>=1 only non-solid blocks reachable
    cur = want.copy()
    for it in range(cfg.n_prop):
        new = cur.copy()
        for b in range(e - s):
            if not cur[b] and (not solid[b] or it == 0):
                if any(v >= 0 and cur[v] for v in nb[b]):
                    new[b] = True
        cur = new
    assert np.array_equal((g.bflags[s:e] & 8) > 0, cur)


def test_boundary_brute_force(O, c1):
    """boundary set equals a brute-force neighbour scan."""
    m, cfg, r = c1
    g = r.grid
    L = g.n_levels - 1
    s, e = g.level_range(L)
    n = cfg.bins(L)[0] * 4
    dense = np.full((n + 2, n + 2, n + 2), -1, dtype=np.int8)  # [x, y, z], 1-cell pad
    t = np.arange(64)
    gi = 4 * g.coords[s:e, None, :3] + np.stack([t & 3, (t >> 2) & 3, t >> 4], 1)[None] + 1
    gi = gi.reshape(-1, 3)
    dense[gi[:, 0], gi[:, 1], gi[:, 2]] = g.masks[s:e].reshape(-1)
    mk = dense[gi[:, 0], gi[:, 1], gi[:, 2]]
    nb_solid = np.zeros(len(gi), dtype=bool)
    for c in D3Q27_C[1:]:
        nb_solid |= dense[gi[:, 0] + c[0], gi[:, 1] + c[1], gi[:, 2] + c[2]] == 1
    cand = (mk == 0) | (mk == 5)
    assert np.array_equal((mk == 5)[cand], nb_solid[cand])
    assert (mk == 5).sum() > 1000


def _ray_tri(o, c, tri):
    """Independent Moller-Trumbore in long double: parameter t along c."""
    o = o.astype(np.longdouble)
    c = c.astype(np.longdouble)
    v0, v1, v2 = (tri[k * 3:k * 3 + 3].astype(np.longdouble) for k in range(3))
    e1, e2 = v1 - v0, v2 - v0
    p = np.cross(c, e2)
    det = e1 @ p
    if abs(det) < 1e-30:
        return None
    s = o - v0
    u = (s @ p) / det
    qv = np.cross(s, e1)
    w = (c @ qv) / det
    t = (e2 @ qv) / det
    tol = 1e-9
    if u < -tol or w < -tol or u + w > 1 + tol:
        return None
    return float(t)


def test_link_lengths_independent(O, c1):
    """q = d/dx matches an independent ray-triangle oracle (SPEC.md:345 on
    the faceted sphere) and fluid directions are exactly -1."""
    m, cfg, r = c1
    g = r.grid
    L = g.n_levels - 1
    dx = cfg.dx(L)
    s, e = g.level_range(L)
    rng = np.random.default_rng(0)
    mapped = np.where(r.contraction_map[s:e] >= 0)[0]
    fc = m.faces_coord.reshape(-1, 3, 3)
    flo, fhi = fc.min(axis=1), fc.max(axis=1)
    checked = 0
    for bi in rng.choice(mapped, size=min(40, len(mapped)), replace=False):
        b = s + bi
        slot = r.contraction_map[b]
        co = g.coords[b, :3]
        for t in range(0, 64, 3):
            if g.masks[b, t] != 5:
                continue
            x = (4 * co + np.array([t & 3, (t >> 2) & 3, t >> 4]) + 0.5) * dx
            near = np.where(np.all(flo <= x + 2 * dx, axis=1) & np.all(fhi >= x - 2 * dx, axis=1))[0]
            for q in range(1, 27):
                c = D3Q27_C[q].astype(np.float64)
                best = np.inf
                for f in near:
                    tt = _ray_tri(x, c, m.faces_coord[f])
                    if tt is not None and 0 < tt <= dx:
                        best = min(best, tt)
                got = r.lengths[slot, q, t]
                if best == np.inf:
                    assert got == -1.0 or got * dx <= 1e-7 + 0 * got
                else:
                    assert abs(got - best / dx) < 1e-6, (got, best / dx)
                checked += 1
    assert checked > 100


def test_flat_wall_q(O):
    """plane wall between x_b and its solid neighbour:
    q = (x_w - x_b)/dx exactly."""
    xw = 0.5 + 0.3 / 32
    lo, hi = np.array([xw, 0.2, 0.2]), np.array([0.8, 0.8, 0.8])
    v = np.array([[x, y, z] for z in (lo[2], hi[2]) for y in (lo[1], hi[1]) for x in (lo[0], hi[0])])
    quads = [[0, 2, 3, 1], [4, 5, 7, 6], [0, 1, 5, 4], [2, 6, 7, 3], [0, 4, 6, 2], [1, 3, 7, 5]]
    faces = [[qq[0], qq[1], qq[2]] for qq in quads] + [[qq[0], qq[2], qq[3]] for qq in quads]
    m = TriangleMesh(v, faces)
    cfg = EmbedConfig(n_x=32, l_max=1)
    r = O.embed(m.faces_coord, m.normals, cfg, 600)
    g = r.grid
    dx = cfg.dx(0)
    found = 0
    for b in range(g.n_used):
        slot = r.contraction_map[b]
        if slot < 0:
            continue
        for t in range(64):
            gi = 4 * g.coords[b, :3] + np.array([t & 3, (t >> 2) & 3, t >> 4])
            x = (gi + 0.5) * dx
            if g.masks[b, t] == 5 and x[0] < xw and xw - x[0] < dx and 0.25 < x[1] < 0.75 and 0.25 < x[2] < 0.75:
                assert r.lengths[slot, 1, t] == np.float32((xw - x[0]) / dx)
                assert r.lengths[slot, 2, t] == -1.0
                found += 1
    assert found > 50


def test_filter_and_thread_invariance(O):
    """SPEC.md:552 acceptance #4: identical with filtering on/off and across
    thread counts {1, 4, 8}."""
    m = translate(make_torus(60, 30), (0.004, 0.002, -0.003))
    cfg = EmbedConfig(n_x=32, l_max=3)
    cap = 60000
    outs = []
    for thr, filt in ((8, True), (1, True), (4, False)):
        O.set_threads(thr)
        outs.append(O.embed(m.faces_coord, m.normals, cfg, cap, use_filter=filt))
    O.set_threads(os.cpu_count() or 1)
    a = outs[0]
    for b in outs[1:]:
        for k in ("coords", "nbr", "nbr_child", "child", "bflags", "masks"):
            assert np.array_equal(getattr(a.grid, k)[:a.grid.n_used], getattr(b.grid, k)[:b.grid.n_used])
        assert np.array_equal(a.lengths, b.lengths)


def test_refine_faces_cap():
    m = make_icosphere((0.5, 0.5, 0.5), 0.5, 1)
    ls = l_spec_bound((1, 1, 1), 2, 3, 16)
    r = refine_faces(m, ls)
    assert r.max_edge_lengths().max() < ls
    assert abs(r.face_areas().sum() - m.face_areas().sum()) < 1e-12
    assert refine_faces(r, ls) is r  # identity when already fine


@pytest.mark.parametrize("case", ["ico1", "torus", "rand", "dup", "mixed"])
def test_refine_faces_reference_order(case):
    """refine_faces reproduces the reference's face AND vertex numbering
    (geometry.py:355-403, depth-first stack walk), pinned by vectors generated
    from the reference (tests/golden/make_refine_golden.py)."""
    z = np.load(os.path.join(GOLD, "refine_golden.npz"))
    r = refine_faces(TriangleMesh(z[case + "_V"], z[case + "_F"]), float(z[case + "_l"]))
    assert np.array_equal(r.faces_indexed, z[case + "_RF"])
    assert np.array_equal(r.vertices, z[case + "_RV"])


def test_torus_generator():
    m = make_torus(40, 20)
    assert m.n_faces == 1600
    cen = m.faces_coord.reshape(-1, 3, 3).mean(axis=1) - 0.5
    ring = cen.copy()
    ring[:, 2] = 0
    ring = 0.25 * ring / np.linalg.norm(ring, axis=1, keepdims=True)
    assert np.all(np.sum((cen - ring) * m.normals, axis=1) > 0)  # outward
