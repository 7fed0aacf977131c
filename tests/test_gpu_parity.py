"""GPU parity tests: every CUDA stage against the CPU oracle on the same inputs
(bit-exact for masks, flags, topology, bins; link lengths <= 1e-5 relative, the
north-star FP32 tolerance), called through the C-ABI via the package API."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2512_01251_b200 import EmbedConfig, make_icosphere, make_torus  # noqa: E402
from paper_2512_01251_b200 import binning, forest, voxelizer  # noqa: E402
from paper_2512_01251_b200.datatypes import ForestGrid, as_device_mesh  # noqa: E402
from paper_2512_01251_b200.mesh import translate  # noqa: E402
from paper_2512_01251_b200.voxelizer import EmbedEngine  # noqa: E402

LINK_RTOL = 1e-5  # north star: cut-link distances within 1e-5 relative (FP32)


@pytest.fixture(scope="module")
def O(oracle_mod):
    return oracle_mod


@pytest.fixture(scope="module")
def sphere():
    return make_icosphere((0.5, 0.5, 0.5), 0.5, 4)


@pytest.fixture(scope="module")
def torus():
    return translate(make_torus(70, 40), (0.0031, -0.0017, 0.0023))


def grid_equal(gpu, ref, n=None, keys=("coords", "nbr", "nbr_child", "child", "bflags", "masks")):
    n = ref.n_used if n is None else n
    for k in keys:
        a = gpu[k][:n]
        b = getattr(ref, k)[:n]
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)
            raise AssertionError(f"{k}: {len(bad)} mismatches, first at {bad[:5].tolist()}")


def check_links(lg, lr):
    assert lg.shape == lr.shape
    neg = lr < 0
    assert np.array_equal(lg < 0, neg), "-1 pattern differs"
    assert np.all(lg[neg] == -1.0)
    if (~neg).any():
        rel = np.abs(lg[~neg] - lr[~neg]) / np.abs(lr[~neg])
        assert rel.max() <= LINK_RTOL, rel.max()


def test_sat_golden():
    import ctypes as C
    from paper_2512_01251_b200 import _lib
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "sat_golden.npz"))
    lib = _lib.require_cuda()
    tri = torch.from_numpy(z["tri"]).cuda()
    box = torch.from_numpy(z["box"]).cuda()
    out = torch.empty(len(z["out"]), dtype=torch.uint8, device="cuda")
    _lib.check(lib.vf_sat_batch(_lib.ptr(tri), _lib.ptr(box), len(out), _lib.ptr(out),
                                _lib.stream_ptr()))
    got = out.cpu().numpy().astype(bool)
    assert np.array_equal(got, z["out"]), int((got != z["out"]).sum())


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("L", [0, 1, 2])
def test_ray_indicators(O, sphere, mode, L):
    cfg = EmbedConfig(n_x=32, l_max=3)
    got = binning.compute_ray_indicators(sphere, L, mode, cfg).cpu().numpy()
    ref = O.ray_indicators(sphere.faces_coord, sphere.normals, cfg, L, mode)
    assert np.array_equal(got, ref)


def test_compact(O):
    rng = np.random.default_rng(0)
    for n in (0, 1, 5, 4096, 4097, 100003):
        ind = (rng.random(n) < 0.3).astype(np.uint8)
        fm = binning.compact_filtered_faces(torch.from_numpy(ind).cuda())
        assert np.array_equal(fm.compact_map.cpu().numpy(), O.compact(ind))
    fm = binning.compact_filtered_faces(torch.tensor([0, 1, 1, 0, 1], dtype=torch.uint8))
    assert fm.compact_map.cpu().tolist() == [1, 2, 4]


@pytest.mark.parametrize("L", [0, 2])
def test_bin_pairs_and_assemble(O, torus, L):
    cfg = EmbedConfig(n_x=32, l_max=3)
    ind = O.ray_indicators(torus.faces_coord, torus.normals, cfg, L, 0)
    fmap_np = O.compact(ind)
    pb_r, pf_r = O.bin_pairs(torus.faces_coord, fmap_np, cfg, L)
    fm = binning.FilterMap(None, torch.from_numpy(fmap_np).cuda())
    pb, pf = binning.compute_bin_pairs(torus, fm, L, cfg)
    assert np.array_equal(pb.cpu().numpy(), pb_r)
    assert np.array_equal(pf.cpu().numpy(), pf_r)
    bl = binning.assemble_bins((pb, pf), cfg.n_bins(L), L, cfg.bins(L))
    c, o, f = bl.to_numpy()
    cr, orr, fr = O.assemble(pb_r, pf_r, cfg.n_bins(L))
    assert np.array_equal(c, cr) and np.array_equal(o, orr) and np.array_equal(f, fr)


def test_assemble_spec_example():
    # [(2,f0),(0,f1),(2,f3)] -> counts{0:1,2:2}, offsets{0:0,2:1}, [f1,f0,f3]
    pb = torch.tensor([2, 0, 2], dtype=torch.int32)
    pf = torch.tensor([0, 1, 3], dtype=torch.int32)
    bl = binning.assemble_bins((pb, pf), 4)
    c, o, f = bl.to_numpy()
    assert c.tolist() == [1, 0, 2, 0] and o[0] == 0 and o[2] == 1 and f.tolist() == [1, 0, 3]


def test_assemble_large_bins(O):
    # long bins exercise the CTA rank sort; random emission order
    rng = np.random.default_rng(3)
    n_bins, P = 64, 60000
    pb = rng.integers(0, 8, size=P).astype(np.int32) * 8
    pf = rng.permutation(P).astype(np.int32)
    bl = binning.assemble_bins((torch.from_numpy(pb), torch.from_numpy(pf)), n_bins)
    c, o, f = bl.to_numpy()
    cr, orr, fr = O.assemble(pb, pf, n_bins)
    assert np.array_equal(c, cr) and np.array_equal(o, orr)
    for b in range(n_bins):  # within a bin: ascending face ids
        assert np.array_equal(np.sort(fr[orr[b]:orr[b] + cr[b]]), f[o[b]:o[b] + c[b]])


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("use_filter", [True, False])
def test_build_level(O, sphere, mode, use_filter):
    cfg = EmbedConfig(n_x=32, l_max=3)
    for L in range(3):
        bl = binning.build_level(sphere, L, cfg, mode, use_filter)
        c, o, f = bl.to_numpy()
        cr, orr, fr = O.build_bins(sphere.faces_coord, sphere.normals, cfg, L, mode, use_filter)
        assert np.array_equal(c, cr) and np.array_equal(o, orr) and np.array_equal(f, fr)


def _oracle_state_through(O, mesh, cfg, upto_level, stage):
    """Run the oracle pipeline and return the grid state just before `stage`
    at level `upto_level`."""
    cap = cfg.block_capacity(mesh.face_areas().sum())
    g = O.init_forest(cfg, cap)
    fc, nrm = mesh.faces_coord, mesh.normals
    for L in range(cfg.l_max):
        bins = O.build_bins(fc, nrm, cfg, L)
        if L == upto_level and stage == "voxelize":
            return g, bins
        O.voxelize_level(g, cfg, L, bins, fc, nrm)
        if L == upto_level and stage == "propagate+":
            return g, bins
        O.propagate(g, cfg, L, +1)
        if L == upto_level and stage == "propagate-":
            return g, bins
        if L > 0:
            O.propagate(g, cfg, L, -1)
        if L == upto_level and stage == "finalize":
            return g, bins
        O.finalize(g, cfg, L)
        if L == upto_level and stage == "mark":
            return g, bins
        if L == cfg.l_max - 1:
            return g, bins
        O.mark(g, cfg, L)
        if L == upto_level and stage == "adapt":
            return g, bins
        O.adapt(g, cfg, L)
    return g, None


def _gpu_grid(cfg, g):
    return ForestGrid.from_numpy(cfg, dict(coords=g.coords, nbr=g.nbr, nbr_child=g.nbr_child,
                                           child=g.child, bflags=g.bflags, masks=g.masks,
                                           level_start=g.level_start, n_levels=g.n_levels))


@pytest.mark.parametrize("L", [0, 1, 2])
def test_stage_voxelize(O, torus, L):
    cfg = EmbedConfig(n_x=32, l_max=3)
    g, bins = _oracle_state_through(O, torus, cfg, L, "voxelize")
    gg = _gpu_grid(cfg, g)
    bl = binning.BinLevel(L, cfg.bins(L), *(torch.from_numpy(a).cuda() for a in (bins[2], bins[0], bins[1])))
    voxelizer.partial_surface_voxelize(gg, L, bl, torus)
    O.voxelize_level(g, cfg, L, bins, torus.faces_coord, torus.normals)
    grid_equal(gg.to_numpy(), g)


@pytest.mark.parametrize("L", [0, 1, 2])
@pytest.mark.parametrize("stage", ["propagate+", "propagate-", "finalize"])
def test_stage_propagate(O, torus, L, stage):
    if stage == "propagate-" and L == 0:
        pytest.skip("no -x pass on the root grid (PAPER.md:770)")
    cfg = EmbedConfig(n_x=32, l_max=3)
    g, _ = _oracle_state_through(O, torus, cfg, L, stage)
    gg = _gpu_grid(cfg, g)
    if stage == "propagate+":
        voxelizer.propagate_external(gg, L, +1)
        O.propagate(g, cfg, L, +1)
    elif stage == "propagate-":
        voxelizer.propagate_external(gg, L, -1)
        O.propagate(g, cfg, L, -1)
    else:
        voxelizer.finalize_masks(gg, L)
        O.finalize(g, cfg, L)
    grid_equal(gg.to_numpy(), g)


@pytest.mark.parametrize("L", [0, 1])
def test_stage_mark_adapt(O, torus, L):
    cfg = EmbedConfig(n_x=32, l_max=3)
    g, _ = _oracle_state_through(O, torus, cfg, L, "mark")
    gg = _gpu_grid(cfg, g)
    voxelizer.mark_near_wall_refinement(gg, L)
    O.mark(g, cfg, L)
    grid_equal(gg.to_numpy(), g)
    forest.adapt(gg)
    O.adapt(g, cfg, L)
    assert gg.n_levels == g.n_levels
    grid_equal(gg.to_numpy(), g)


def test_stage_boundary_tables_links(O, torus):
    cfg = EmbedConfig(n_x=32, l_max=3)
    g, _ = _oracle_state_through(O, torus, cfg, 2, "mark")  # finest level finalized
    gg = _gpu_grid(cfg, g)
    counts = voxelizer.identify_boundary_cells(gg)
    bc = O.boundary(g, cfg)
    grid_equal(gg.to_numpy(), g)
    n = g.n_used
    assert np.array_equal(counts.cpu().numpy()[:n], bc[:n])
    table = voxelizer.build_boundary_tables(gg)           # SPEC.md:328 signature
    nb, cmap = O.tables(g, bc)
    assert table.n_b == nb
    assert np.array_equal(table.contraction_map.cpu().numpy(), cmap)
    md = O.build_bins(torus.faces_coord, torus.normals, cfg, 2, mode=1)
    lr = O.link_lengths(g, cfg, cmap, nb, md, torus.faces_coord, torus.normals)
    t2 = voxelizer.compute_link_lengths(gg, None, torus)   # SPEC.md:337 signature
    assert t2 is table
    check_links(table.lengths.cpu().numpy(), lr)
    # explicit counts / table (the extended form) and counts from the masks
    gg.bcount = None
    t3 = voxelizer.build_boundary_tables(gg)
    assert t3.n_b == nb and np.array_equal(t3.contraction_map.cpu().numpy(), cmap)
    voxelizer.compute_link_lengths(gg, None, torus, voxelizer.build_boundary_tables(gg, counts))
    check_links(gg.table.lengths.cpu().numpy(), lr)


def test_block_of_point_exhaustive():
    """1,000 random points, block_of_point vs an exhaustive
    containment scan over the leaves and over each level; SPEC.md:244 ties
    at block faces go to the lower index."""
    from paper_2512_01251_b200.forest import block_of_point
    cfg = EmbedConfig(n_x=32, l_max=3)
    grid, _ = EmbedEngine(make_torus(60, 30), cfg).run()
    g = grid.to_numpy()
    n = int(g["level_start"][grid.n_levels])
    co, child = g["coords"][:n], g["child"][:n]
    h = 4.0 * cfg.dx0 / 2.0 ** co[:, 3]
    lo = co[:, :3] * h[:, None]
    hi = lo + h[:, None]
    rng = np.random.default_rng(7)
    for p in rng.random((1000, 3)):
        inside = np.all((lo <= p) & (p <= hi), axis=1)
        leaves = np.nonzero(inside & (child < 0))[0]
        assert len(leaves) == 1
        assert block_of_point(grid, p) == leaves[0]
        for L in range(grid.n_levels):
            at = np.nonzero(inside & (co[:, 3] == L))[0]
            got = block_of_point(grid, p, L)
            assert (got is None and len(at) == 0) or (len(at) == 1 and got == at[0])
    # a point on a root-block corner goes to the lower-index block
    h0 = 4.0 * cfg.dx0
    b = block_of_point(grid, (h0, h0, h0), 0)
    assert tuple(co[b, :3]) == (0, 0, 0)


def test_embed_geometry_cached(O, torus):
    """SPEC.md:346 embed_geometry: the engine (and its graph) is reused for
    the same mesh + config; results equal the oracle; copy=True detaches."""
    from paper_2512_01251_b200.voxelizer import embed_geometry, _ENGINES
    cfg = EmbedConfig(n_x=32, l_max=3)
    g1, t1 = embed_geometry(None, torus, cfg)
    g2, t2 = embed_geometry(None, torus, cfg)
    assert g1 is g2 and t2.lengths.data_ptr() == t1.lengths.data_ptr()
    g3, t3 = embed_geometry(None, torus, cfg, copy=True)
    assert t3.lengths.data_ptr() != t1.lengths.data_ptr()
    ref = O.embed(torus.faces_coord, torus.normals, cfg, capacity=g3.capacity)
    grid_equal(g3.to_numpy(), ref.grid)
    check_links(t3.lengths.cpu().numpy(), ref.lengths)
    other = make_icosphere((0.5, 0.5, 0.5), 0.5, 3)
    g4, _ = embed_geometry(None, other, cfg)
    assert g4 is not g1


def _embed_compare(O, mesh, cfg, use_filter=True):
    eng = EmbedEngine(mesh, cfg)
    grid, table = eng.run(use_filter=use_filter)
    torch.cuda.synchronize()
    ref = O.embed(mesh.faces_coord, mesh.normals, cfg, capacity=grid.capacity,
                  use_filter=use_filter)
    gn = grid.to_numpy()
    assert grid.n_levels == ref.grid.n_levels
    assert np.array_equal(gn["level_start"], ref.grid.level_start)
    grid_equal(gn, ref.grid)
    assert table.n_b == ref.n_b
    assert np.array_equal(table.contraction_map.cpu().numpy()[:ref.grid.n_used], ref.contraction_map)
    check_links(table.lengths.cpu().numpy(), ref.lengths)
    return eng, grid, table


def test_embed_c1_sphere(O):
    """C1: icosphere 20,480 faces, N_x=64, L_max=3."""
    mesh = make_icosphere((0.5, 0.5, 0.5), 0.5, 5)
    _embed_compare(O, mesh, EmbedConfig(n_x=64, l_max=3))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_embed_translated_torus(O, seed):
    rng = np.random.default_rng(seed)
    mesh = translate(make_torus(120, 60), rng.random(3) / 64.0 - 1 / 128.0)
    _embed_compare(O, mesh, EmbedConfig(n_x=32, l_max=4))


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
def test_embed_c2_robustness_translations(O, seed):
    """SURVEY.md §8d robustness variants: the C2 mesh rigidly translated by
    np.random.default_rng(seed).random(3) * dx_0 (offsets in [0, dx_0)^3),
    seeds 0-4, at the C2 configuration."""
    cfg = EmbedConfig(n_x=64, l_max=4)
    mesh = translate(make_torus(280, 200), np.random.default_rng(seed).random(3) * cfg.dx0)
    _embed_compare(O, mesh, cfg)


def test_embed_filter_invariance_and_determinism(O, torus):
    cfg = EmbedConfig(n_x=32, l_max=3)
    eng = EmbedEngine(torus, cfg)
    g1, t1 = eng.run(use_filter=True)
    a = g1.to_numpy()
    la = t1.lengths.cpu().numpy().copy()
    g2, t2 = eng.run(use_filter=False)
    b = g2.to_numpy()
    for k in ("coords", "nbr", "nbr_child", "child", "bflags", "masks", "level_start"):
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(la, t2.lengths.cpu().numpy())
    g3, t3 = eng.run()
    c = g3.to_numpy()
    for k in ("masks", "nbr"):
        assert np.array_equal(a[k], c[k])
    assert np.array_equal(la, t3.lengths.cpu().numpy())


def test_capacity_error():
    from paper_2512_01251_b200 import CapacityError
    mesh = make_icosphere((0.5, 0.5, 0.5), 0.5, 3)
    cfg = EmbedConfig(n_x=32, l_max=3)
    with pytest.raises(CapacityError):
        EmbedEngine(mesh, cfg, capacity=600).run()


def test_smoke():
    import __graft_entry__
    __graft_entry__.smoke()


# ---------------------------------------------------------------------------
# grid-aligned degeneracies: faces through lattice nodes, edges on lattice
# lines, vertices on cell centres -- the cases where the FP32 classifiers of
# k_voxelize / k_links must hand the decision to the exact FP64 SAT.

def _box_mesh(lo, hi, n, rot_z=0.0):
    """Closed axis-aligned box [lo, hi]^3 (n x n quads per side, 2 triangles
    each, outward), optionally rotated about the z axis through its centre."""
    from paper_2512_01251_b200.mesh import TriangleMesh
    lo, hi = np.asarray(lo, float), np.asarray(hi, float)
    verts, faces = [], []
    t = np.linspace(0.0, 1.0, n + 1)
    for axis in range(3):
        for side in (0, 1):
            a, b = [d for d in range(3) if d != axis]
            base = len(verts)
            for i in range(n + 1):
                for j in range(n + 1):
                    p = np.empty(3)
                    p[axis] = hi[axis] if side else lo[axis]
                    p[a] = lo[a] + t[i] * (hi[a] - lo[a])
                    p[b] = lo[b] + t[j] * (hi[b] - lo[b])
                    verts.append(p)
            for i in range(n):
                for j in range(n):
                    v00 = base + i * (n + 1) + j
                    v10, v01, v11 = v00 + (n + 1), v00 + 1, v00 + n + 2
                    # (a, b, axis) right-handed?  orient so the normal points out
                    right = (b - a) % 3 == 1
                    out = (side == 1) == right
                    if out:
                        faces += [[v00, v10, v11], [v00, v11, v01]]
                    else:
                        faces += [[v00, v11, v10], [v00, v01, v11]]
    V = np.array(verts)
    # weld duplicate corner/edge vertices so the mesh is closed
    key = np.round(V * 2**40).astype(np.int64)
    _, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
    F = first[inv.reshape(-1)][np.array(faces)]
    if rot_z:
        c = 0.5 * (lo + hi)
        cs, sn = np.cos(rot_z), np.sin(rot_z)
        R = np.array([[cs, -sn, 0], [sn, cs, 0], [0, 0, 1]])
        V = (V - c) @ R.T + c
    m = TriangleMesh(V, F)
    # outward check: signed volume > 0
    v = V[F]
    vol = np.einsum("ij,ij->i", v[:, 0], np.cross(v[:, 1], v[:, 2])).sum() / 6.0
    if vol < 0:
        m = TriangleMesh(V, F[:, ::-1])
    return m


@pytest.mark.parametrize("case", ["nodes", "faces", "rotated"])
def test_embed_grid_aligned(O, case):
    cfg = EmbedConfig(n_x=32, l_max=3)
    dxf = 1.0 / 32 / 4  # finest cell size
    if case == "nodes":      # box faces through finest-level cell centres
        lo, hi = 0.3 + 0.5 * dxf, 0.7 + 0.5 * dxf
        mesh = _box_mesh([lo] * 3, [hi] * 3, 8)
    elif case == "faces":    # box faces on cell boundaries, vertices on lattice corners
        mesh = _box_mesh([0.25] * 3, [0.75] * 3, 16)
    else:                    # 45 degrees about z: diagonal links graze edges
        mesh = _box_mesh([0.3 + 0.5 * dxf] * 3, [0.7 + 0.5 * dxf] * 3, 8, rot_z=np.pi / 4)
    _embed_compare(O, mesh, cfg)


def test_links_band_overflow_fallback(O, torus):
    """Band list capacity 0: every undecided candidate overflows and the
    fallback pass redoes every face inline -- the LUT must not change."""
    from paper_2512_01251_b200 import _lib
    lib = _lib.require_cuda()
    cfg = EmbedConfig(n_x=32, l_max=3)
    mesh = _box_mesh([0.3 + 0.5 / 128] * 3, [0.7 + 0.5 / 128] * 3, 8, rot_z=np.pi / 4)
    for m in (torus, mesh):
        eng = EmbedEngine(m, cfg, use_graph=False)
        _, t1 = eng.run()
        a = t1.lengths.cpu().numpy().copy()
        old = lib.vf_set_link_band_cap(0)
        try:
            _, t2 = eng.run()
            b = t2.lengths.cpu().numpy()
        finally:
            lib.vf_set_link_band_cap(old)
        assert np.array_equal(a, b)


@pytest.mark.parametrize("small_ext", [-1.0, 0.5, 1e9])
def test_links_small_face_split(O, torus, small_ext):
    """The thread-per-face enumeration of small faces and the warp-flattened
    one of large faces are interchangeable: every face through either kernel
    (or a mixed split) gives the oracle's LUT."""
    from paper_2512_01251_b200 import _lib
    lib = _lib.require_cuda()
    cfg = EmbedConfig(n_x=32, l_max=3)
    mesh = _box_mesh([0.3 + 0.5 / 128] * 3, [0.7 + 0.5 / 128] * 3, 8, rot_z=np.pi / 4)
    old = lib.vf_set_link_small_ext(small_ext)
    try:
        for m in (torus, mesh, make_torus(300, 120)):
            _embed_compare(O, m, cfg)
    finally:
        lib.vf_set_link_small_ext(old)


def test_sparse_rows(O, torus):
    """Alg. 5 over the sparse row order (vf_rows.cu): short rows, rows of
    B_L = 256, and long x-runs spanning several 32-block chunks (a slab whose
    faces parallel to x refine whole rows) give the oracle's masks."""
    _embed_compare(O, torus, EmbedConfig(n_x=32, l_max=3))
    _embed_compare(O, make_icosphere((0.5, 0.5, 0.5), 0.5, 4), EmbedConfig(n_x=64, l_max=3))
    _embed_compare(O, make_torus(300, 120), EmbedConfig(n_x=64, l_max=5))  # B_L = 256 rows
    slab = _box_mesh([0.03 + 0.5 / 512, 0.41 + 0.3 / 512, 0.44 + 0.7 / 512], [0.97 - 0.5 / 512, 0.6, 0.55], 24)
    _embed_compare(O, slab, EmbedConfig(n_x=64, l_max=4))


def test_serial_links_identical(torus):
    """The measurement schedule (enumeration serial on the main stream) gives
    the same LUT and cut-link map as the overlapped production schedule."""
    from paper_2512_01251_b200 import _lib
    lib = _lib.require_cuda()
    eng = EmbedEngine(torus, EmbedConfig(n_x=32, l_max=3), use_graph=False)
    g1, t1 = eng.run(timed=True)
    a, ca = t1.lengths.cpu().numpy().copy(), t1.contraction_map.cpu().numpy().copy()
    old = lib.vf_set_serial_links(1)
    try:
        _, t2 = eng.run(timed=True)
        b, cb = t2.lengths.cpu().numpy(), t2.contraction_map.cpu().numpy()
        assert eng.link_kernel_ms() > 0
    finally:
        lib.vf_set_serial_links(old)
    assert np.array_equal(a, b) and np.array_equal(ca, cb)


def test_cli_voxelize(tmp_path):
    """CLI voxelize: one VTK per level, masks equal to the engine's, summary."""
    import json
    from paper_2512_01251_b200 import cli
    from paper_2512_01251_b200.vtk import read_vtk_cell_data
    rc = cli.main(["voxelize", "--primitive", "sphere", "--nx", "16", "--lmax", "2", "--out", str(tmp_path)])
    assert rc == 0
    summary = json.load(open(tmp_path / "summary.json"))
    assert summary["files"] == ["level_0.vtk", "level_1.vtk"] and summary["links"] > 0
    grid, table = EmbedEngine(make_icosphere((0.5, 0.5, 0.5), 0.5, 4), EmbedConfig(n_x=16, l_max=2)).run()
    g = grid.to_numpy()
    for L in range(2):
        s, e = int(g["level_start"][L]), int(g["level_start"][L + 1])
        d = read_vtk_cell_data(str(tmp_path / f"level_{L}.vtk"))
        assert np.array_equal(d["mask"], g["masks"][s:e].reshape(-1))


# ---------------------------------------------------------------------------
# configuration edge cases: code paths the default configs never take

def _open_patch():
    """A small open surface (two triangles) partly outside the domain."""
    from paper_2512_01251_b200.mesh import TriangleMesh
    V = np.array([[0.30, 0.40, 0.55], [0.80, 0.35, 0.60], [0.45, 0.85, 0.40], [1.20, 0.90, 0.50]])
    return TriangleMesh(V, np.array([[0, 1, 2], [1, 3, 2]]))


@pytest.mark.parametrize("case", ["nx48_nonpow2", "domain_2x1x1", "eps0", "no_filter_torus",
                                  "open_patch", "lmax1", "nspec1", "bincap"])
def test_embed_config_edges(O, case):
    torus = translate(make_torus(60, 30), (0.0021, -0.0013, 0.0017))
    if case == "nx48_nonpow2":      # dx = 1/48: inexact 1/dx, widened ranges
        mesh, cfg = torus, EmbedConfig(n_x=48, l_max=3)
    elif case == "domain_2x1x1":    # non-cubic domain, mesh off-centre
        mesh, cfg = translate(torus, (0.6, 0.0, 0.0)), EmbedConfig(n_x=32, l_max=3, domain=(2.0, 1.0, 1.0))
    elif case == "eps0":            # eps_slab = 0: the link fast path is disabled
        mesh, cfg = torus, EmbedConfig(n_x=32, l_max=3, eps_slab=0.0)
    elif case == "no_filter_torus":
        mesh, cfg = torus, EmbedConfig(n_x=32, l_max=3, use_filter=False)
    elif case == "open_patch":      # open surface leaving the domain, refined to l_spec
        from paper_2512_01251_b200.mesh import l_spec_bound, refine_faces
        cfg = EmbedConfig(n_x=32, l_max=3)
        mesh = refine_faces(_open_patch(), l_spec_bound(cfg.domain, cfg.n_spec, cfg.l_max, cfg.nb[0]))
    elif case == "lmax1":           # root level only: no refinement
        mesh, cfg = torus, EmbedConfig(n_x=32, l_max=1)
    elif case == "nspec1":          # N_spec = 1 -> N_lim = 27 pairs / face
        mesh, cfg = torus, EmbedConfig(n_x=32, l_max=3, n_spec=1)
    else:                           # faces above l_spec: the N_lim cap is asserted
        from paper_2512_01251_b200 import BinCapError
        with pytest.raises(BinCapError):
            EmbedEngine(_open_patch(), EmbedConfig(n_x=32, l_max=3)).run()
        return
    _embed_compare(O, mesh, cfg, use_filter=cfg.use_filter)


@pytest.mark.parametrize("case", ["nx48_nonpow2", "domain_2x1x1", "eps0", "open_patch"])
def test_embed_config_edges_small_path(O, case):
    """The same edge configurations with every face through the thread-per-
    face cut-link enumeration (non-power-of-two dx, non-cubic domain, no
    fast path, faces leaving the domain)."""
    from paper_2512_01251_b200 import _lib
    lib = _lib.require_cuda()
    old = lib.vf_set_link_small_ext(1e9)
    try:
        test_embed_config_edges(O, case)
    finally:
        lib.vf_set_link_small_ext(old)


def test_embed_c2_bench_config(O):
    """The bench workload itself (C2: 112,000-face torus, N_x=64, L_max=4)
    against the oracle, end to end."""
    _embed_compare(O, make_torus(280, 200), EmbedConfig(n_x=64, l_max=4))


def test_embed_c4_flagship(O):
    """C4 (7,200,000-face torus, L_max=5: the north-star mesh) against the
    oracle, end to end -- also exercises the eager (>1M faces) launch path."""
    _embed_compare(O, make_torus(3000, 1200), EmbedConfig(n_x=64, l_max=5))


def test_ctx_create_destroy(O, torus):
    """vf_ctx_create / vf_ctx_destroy: the context owns the
    device's side streams; an embed after destroy recreates them."""
    from paper_2512_01251_b200 import _lib
    lib = _lib.require_cuda()
    ctx = lib.vf_ctx_create(0, None)
    assert ctx and lib.vf_ctx_device(ctx) == 0
    cfg = EmbedConfig(n_x=32, l_max=3)
    _embed_compare(O, torus, cfg)
    assert lib.vf_ctx_destroy(ctx) == 0
    _embed_compare(O, torus, cfg)


def test_link_stats(torus):
    """vf_embed_link_stats: counters of the last embed's cut-link pass."""
    eng = EmbedEngine(torus, EmbedConfig(n_x=32, l_max=3), use_graph=False)
    _, table = eng.run()
    st = eng.link_stats()
    assert st["lines"] > 0 and st["lines"] <= st["line_cap"]
    assert st["overflow_faces"] == 0 and 0 <= st["band"] <= st["band_cap"]
    assert 0 <= st["large_faces"] <= torus.n_faces
    assert int((table.lengths >= 0).sum()) > 0


def test_kernel_timer(O, torus):
    """vf_ktimer_*: per-kernel times of one serial eager embed; the embed it
    times gives the oracle's result (same kernels, one stream)."""
    cfg = EmbedConfig(n_x=32, l_max=3)
    eng = EmbedEngine(torus, cfg)
    eng.run()
    kt = eng.kernel_times()
    assert "k_voxelize" in kt and "k_pairs" in kt and kt["k_voxelize"][0] == cfg.l_max
    assert all(c > 0 and ms >= 0 for c, ms in kt.values())
    ref = O.embed(torus.faces_coord, torus.normals, cfg, capacity=eng.grid.capacity)
    grid_equal(eng.grid.to_numpy(), ref.grid)
    tab = eng.run()[1]
    check_links(tab.lengths.cpu().numpy(), ref.lengths)


def test_indexed_e2e_path(O, torus):
    """The serving path from the indexed mesh: vf_pack_indexed's face records
    and normals are bit-identical to TriangleMesh's (np.cross / norm), and the
    downloaded grid + sparse cut links expand to the oracle's LUT."""
    from paper_2512_01251_b200 import _lib
    from paper_2512_01251_b200.datatypes import lengths_from_sparse
    from paper_2512_01251_b200.errors import MeshError
    lib = _lib.require_cuda()
    cfg = EmbedConfig(n_x=32, l_max=3)
    for mesh in (torus, make_icosphere((0.5, 0.5, 0.5), 0.5, 4)):
        V = torch.from_numpy(np.ascontiguousarray(mesh.vertices)).cuda()
        Fi = torch.from_numpy(np.ascontiguousarray(mesh.faces_indexed, dtype=np.int32)).cuda()
        rec = torch.empty((mesh.n_faces, 12), dtype=torch.float64, device="cuda")
        st = torch.zeros(4, dtype=torch.int32, device="cuda")
        _lib.check(lib.vf_pack_indexed(_lib.ptr(V), V.shape[0], _lib.ptr(Fi), mesh.n_faces, _lib.ptr(rec),
                                       _lib.ptr(st), _lib.stream_ptr()))
        r = rec.cpu().numpy()
        assert int(st[0]) == 0
        assert np.array_equal(r[:, :9].view(np.uint64), mesh.faces_coord.view(np.uint64))
        assert np.array_equal(r[:, 9:].view(np.uint64), np.ascontiguousarray(mesh.normals).view(np.uint64))
        eng = EmbedEngine(mesh, cfg)
        eng.run()
        verts = torch.from_numpy(np.ascontiguousarray(mesh.vertices)).pin_memory()
        fidx = torch.from_numpy(np.ascontiguousarray(mesh.faces_indexed, dtype=np.int32)).pin_memory()
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        out = None
        for _ in range(2):
            out, h2d, d2h = eng.embed_indexed_async(verts, fidx, out, s_in, s_out)
        torch.cuda.synchronize()
        eng.check_async()
        assert h2d == mesh.vertices.shape[0] * 24 + mesh.n_faces * 12
        ref = O.embed(mesh.faces_coord, mesh.normals, cfg, capacity=eng.grid.capacity)
        host = {k: v.numpy() for k, v in out.items()}
        grid_equal(host, ref.grid, keys=("coords", "nbr", "child", "bflags", "masks"))
        assert np.array_equal(host["contraction_map"], ref.contraction_map)
        check_links(lengths_from_sparse(ref.n_b, host["link_index"], host["link_q"]), ref.lengths)
    # an out-of-range face index latches a mesh error
    bad = np.ascontiguousarray(torus.faces_indexed, dtype=np.int32).copy()
    bad[5, 1] = torus.vertices.shape[0] + 3
    eng = EmbedEngine(torus, cfg)
    eng.run()
    vb = torch.from_numpy(np.ascontiguousarray(torus.vertices)).pin_memory()
    fb = torch.from_numpy(bad).pin_memory()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    eng.embed_indexed_async(vb, fb, None, s_in, s_out)
    torch.cuda.synchronize()
    with pytest.raises(MeshError):
        eng.check_async()
