"""The oracle's interface exchange (oracle/lbm_oracle.c)
on an oracle-embedded sphere: constant fields give constant ghosts for both
orders, trilinear fields are reproduced exactly by linear and cubic
interpolation, tensor-cubic fields by cubic interpolation, wherever the full
stencil lies on non-SOLID coarse cells (SPEC.md:421-425 examples); the
schedule of step_hierarchy advances level L 2^L times per coarse step
(SPEC.md:430-434)."""
import numpy as np
import pytest

from lbm_cases import exact_ghosts, level_cells, poly_field, sphere_case


@pytest.fixture(scope="module")
def case(oracle_mod):
    O = oracle_mod
    mesh, cfg, ref = sphere_case(O, l_max=3, n_x=32, sub=2)
    g = ref.grid
    return O, cfg, g


def _grid_dict(g):
    return dict(coords=np.asarray(g.coords), nbr=np.asarray(g.nbr), masks=np.asarray(g.masks),
                child=np.asarray(g.child))


@pytest.mark.parametrize("kind,order", [("const", 1), ("const", 3), ("linear", 1), ("linear", 3),
                                        ("cubic", 3)])
def test_fill_ghosts_reproduces_polynomials(case, kind, order):
    O, cfg, g = case
    gd = _grid_dict(g)
    ls = np.asarray(g.level_start)
    sc, ec, sf, ef = int(ls[0]), int(ls[1]), int(ls[1]), int(ls[2])
    n0 = 4 * cfg.nb[0]
    fc = poly_field(level_cells(gd, sc, ec), n0, kind)
    ff = np.zeros((27, (ef - sf) * 64), np.float32)
    out = O.lbm_fill_ghosts(gd, sf, ef, sc, ec, fc, None, 0.0, 1.0, order, ff)
    want = poly_field(level_cells(gd, sf, ef), 2 * n0, kind)
    idx = exact_ghosts(gd, sf, ef, sc, ec, order)
    assert len(idx) > 100
    assert np.allclose(out[:, idx], want[:, idx], rtol=0, atol=2e-6)
    ghost = np.asarray(g.masks).reshape(-1, 64)[sf:ef].reshape(-1) == 3
    assert np.all(out[:, ghost] != 0) or kind != "const"  # every ghost got a value
    if kind == "const":
        held = out[:, ghost]
        assert np.allclose(held, want[:, ghost], atol=2e-6)


def test_hierarchy_substep_counts(case):
    O, cfg, g = case
    gd = _grid_dict(g)
    ls = np.asarray(g.level_start)
    ranges = [(int(ls[L]), int(ls[L + 1])) for L in range(len(ls) - 1) if ls[L + 1] > ls[L]]
    from paper_2512_01251_b200.solver import equilibrium
    states = []
    for s, e in ranges:
        n = (e - s) * 64
        states.append(np.ascontiguousarray(equilibrium(np.ones(n), np.zeros((n, 3))).T.astype(np.float32)))
    cmap = np.full(len(gd["coords"]), -1, np.int32)
    out, counts = O.lbm_step_hierarchy(gd, ranges, 4 * cfg.nb[0], cmap, np.zeros(27 * 64, np.float32), states,
                                       0.55, (0.0, 0.0, 0.0), ibb=False, open_x=False)
    assert counts == [2 ** L for L in range(len(ranges))]
    # a closed box at rest stays at rest
    for s0, s1 in zip(states, out):
        assert np.allclose(s0, s1, atol=1e-6)
