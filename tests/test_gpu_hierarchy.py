"""GPU interface exchange and step_hierarchy (csrc/vf_lbm.cu k_lbm_fill_ghosts
/ k_lbm_restrict, solver.LbmHierarchy)
against the oracle (oracle/lbm_oracle.c + oracle.lbm_step_hierarchy) on an
embedded sphere with three levels.  Tolerance: FP32 on the GPU vs FP64 in
the oracle from the same FP32 inputs, |d| <= 2e-6 + 2e-5 |f| per population
for one exchange; one coarse step (7 collide/stream steps, 4 exchanges)
|d| <= 1e-5 + 1e-4 |f|."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from lbm_cases import exact_ghosts, level_cells, perturbed_state, poly_field  # noqa: E402
from paper_2512_01251_b200 import EmbedConfig, make_icosphere  # noqa: E402
from paper_2512_01251_b200.solver import (FlowConfig, LbmHierarchy, LbmLevel, level_taus,  # noqa: E402
                                          neq_factors, step_hierarchy)
from paper_2512_01251_b200.voxelizer import EmbedEngine  # noqa: E402

RTOL, ATOL = 2e-5, 2e-6


@pytest.fixture(scope="module")
def O(oracle_mod):
    return oracle_mod


@pytest.fixture(scope="module")
def emb():
    mesh = make_icosphere((0.5, 0.5, 0.5), 0.4, 3)
    cfg = EmbedConfig(n_x=32, l_max=3)
    eng = EmbedEngine(mesh, cfg, use_graph=False)
    grid, table = eng.run()
    torch.cuda.synchronize()
    return cfg, grid, table


def _close(a, b, rtol=RTOL, atol=ATOL):
    err = np.abs(a - b) - (atol + rtol * np.abs(b))
    assert err.max() <= 0, f"max excess {err.max():.3g}"


def _ranges(grid):
    return [grid.level_range(L) for L in range(grid.n_levels)]


@pytest.mark.parametrize("L", [0, 1])
@pytest.mark.parametrize("order,theta,rescale", [(1, 0.0, False), (3, 0.0, True), (3, 0.5, True), (1, 0.5, True)])
def test_fill_ghosts_matches_oracle(O, emb, L, order, theta, rescale):
    cfg, grid, table = emb
    g = grid.to_numpy()
    h = LbmHierarchy(grid, table, FlowConfig(Re=20.0, u_in=0.04, D_s=16.0), order=order, rescale=rescale)
    (sc, ec), (sf, ef) = grid.level_range(L), grid.level_range(L + 1)
    rng = np.random.default_rng(3 + L)
    old = perturbed_state(g["masks"], sc, ec, rng, u=(0.04, 0, 0))
    new = perturbed_state(g["masks"], sc, ec, rng, u=(0.03, 0.01, 0))
    ff = perturbed_state(g["masks"], sf, ef, rng)
    h.levels[L + 1].state.copy_(torch.from_numpy(ff))
    told, tnew = torch.from_numpy(old).cuda(), torch.from_numpy(new).cuda()
    h.fill_ghosts(L, told, tnew, theta)
    got = h.levels[L + 1].state.cpu().numpy()
    want = O.lbm_fill_ghosts(g, sf, ef, sc, ec, old, new, theta, h.factors[L][0], order, ff)
    _close(got, want)
    ghost = g["masks"].reshape(-1, 64)[sf:ef].reshape(-1) == 3
    assert ghost.sum() > 0 and np.abs(got[:, ghost] - ff[:, ghost]).max() > 0  # ghosts were written
    assert np.array_equal(got[:, ~ghost], ff[:, ~ghost])  # nothing else


@pytest.mark.parametrize("L", [0, 1])
def test_restrict_matches_oracle(O, emb, L):
    cfg, grid, table = emb
    g = grid.to_numpy()
    h = LbmHierarchy(grid, table, FlowConfig(Re=20.0, u_in=0.04, D_s=16.0))
    (sc, ec), (sf, ef) = grid.level_range(L), grid.level_range(L + 1)
    rng = np.random.default_rng(11 + L)
    fc = perturbed_state(g["masks"], sc, ec, rng, u=(0.04, 0, 0))
    ff = perturbed_state(g["masks"], sf, ef, rng, u=(0.02, 0, 0.01))
    h.levels[L].state.copy_(torch.from_numpy(fc))
    h.levels[L + 1].state.copy_(torch.from_numpy(ff))
    h.restrict(L)
    got = h.levels[L].state.cpu().numpy()
    want = O.lbm_restrict(g, sc, ec, sf, ef, ff, h.factors[L][1], fc)
    _close(got, want)
    assert np.abs(got - fc).max() > 0  # covered cells were written


@pytest.mark.parametrize("kind,order", [("const", 3), ("linear", 1), ("linear", 3), ("cubic", 3)])
def test_fill_ghosts_reproduces_polynomials(emb, kind, order):
    """constants for both orders, linear exact for both,
    cubic exact for cubic -- wherever the full stencil is on non-SOLID cells."""
    cfg, grid, table = emb
    g = grid.to_numpy()
    h = LbmHierarchy(grid, table, FlowConfig(), order=order, rescale=False)
    (sc, ec), (sf, ef) = grid.level_range(0), grid.level_range(1)
    n0 = 4 * cfg.nb[0]
    fc = torch.from_numpy(poly_field(level_cells(g, sc, ec), n0, kind)).cuda()
    h.levels[1].state.zero_()
    h.fill_ghosts(0, fc, fc, 0.0)
    got = h.levels[1].state.cpu().numpy()
    want = poly_field(level_cells(g, sf, ef), 2 * n0, kind)
    idx = exact_ghosts(g, sf, ef, sc, ec, order)
    assert len(idx) > 100
    assert np.allclose(got[:, idx], want[:, idx], rtol=0, atol=4e-6)


def test_step_hierarchy_matches_oracle(O, emb):
    cfg, grid, table = emb
    g = grid.to_numpy()
    flow = FlowConfig(Re=20.0, u_in=0.04, D_s=16.0, bc_scheme="IBB")
    h = LbmHierarchy(grid, table, flow, order=3)
    rng = np.random.default_rng(5)
    states = []
    for lv in h.levels:
        f0 = perturbed_state(g["masks"], lv.s, lv.e, rng, u=(0.04, 0, 0))
        lv.state.copy_(torch.from_numpy(f0))
        states.append(f0)
    cmap = np.full(grid.capacity, -1, np.int32)
    cm = table.contraction_map.cpu().numpy()
    cmap[:len(cm)] = cm
    step_hierarchy(h, grid, table, flow)
    want, counts = O.lbm_step_hierarchy(g, _ranges(grid), 4 * cfg.nb[0], cmap, table.lengths.cpu().numpy(),
                                        states, flow.tau, (flow.u_in, 0.0, 0.0), True, True, order=3)
    assert h.substeps == counts == [1, 2, 4]
    for lv, w in zip(h.levels, want):
        _close(lv.state.cpu().numpy(), w, rtol=1e-4, atol=1e-5)


def test_taus_acoustic_scaling(emb):
    cfg, grid, table = emb
    flow = FlowConfig(Re=20.0, u_in=0.04, D_s=16.0)
    t = level_taus(flow.tau, 3)
    assert np.isclose(t[1] - 0.5, 2 * (t[0] - 0.5)) and np.isclose(t[2] - 0.5, 4 * (t[0] - 0.5))
    a, b = neq_factors(t[0], t[1])
    assert np.isclose(a * b, 1.0)


def test_closed_box_rest_is_conserved(emb):
    """mass conserved in a closed SBB box (here: the rest state,
    a fixed point of every level and of the exchange; FP32 state, so the
    bound is 1e-6 relative rather than the FP64 1e-12)."""
    cfg, grid, table = emb
    flow = FlowConfig(Re=20.0, u_in=0.04, D_s=16.0, bc_scheme="SBB", open_x=False)  # u_in sets tau only
    h = LbmHierarchy(grid, None, flow, order=3).init_equilibrium(1.0)
    m0 = h.mass()
    h.step(2)
    assert h.substeps == [2, 4, 8]
    assert abs(h.mass() - m0) <= 1e-6 * m0


def test_single_level_is_a_uniform_step():
    """L_max = 1 -> exactly one uniform-grid step."""
    mesh = make_icosphere((0.5, 0.5, 0.5), 0.4, 2)
    cfg = EmbedConfig(n_x=32, l_max=1)
    grid, table = EmbedEngine(mesh, cfg, use_graph=False).run()
    flow = FlowConfig(Re=20.0, u_in=0.04, D_s=16.0)
    h = LbmHierarchy(grid, table, flow)
    lv = LbmLevel(grid, 0, table, flow)
    g = grid.to_numpy()
    f0 = perturbed_state(g["masks"], lv.s, lv.e, np.random.default_rng(1), u=(0.04, 0, 0))
    h.levels[0].state.copy_(torch.from_numpy(f0))
    lv.state.copy_(torch.from_numpy(f0))
    h.step(1)
    lv.step(1)
    assert torch.equal(h.levels[0].state, lv.state)


def test_graph_replay_equals_eager(emb):
    """The captured two-coarse-step graph (bench C3) computes what step() does."""
    cfg, grid, table = emb
    flow = FlowConfig(Re=20.0, u_in=0.04, D_s=16.0)
    a = LbmHierarchy(grid, table, flow).init_equilibrium(1.0, (0.04, 0, 0))
    b = LbmHierarchy(grid, table, flow).init_equilibrium(1.0, (0.04, 0, 0))
    gr = a.graph()  # a: 2 warm-up coarse steps during capture
    gr.replay()     # + 2
    b.step(4)
    torch.cuda.synchronize()
    for la, lb in zip(a.levels, b.levels):
        assert torch.equal(la.state, lb.state)


def test_cli_simulate(tmp_path):
    """`simulate`: embed + step_hierarchy, force samples and a drag summary."""
    import json
    from paper_2512_01251_b200 import cli
    cfgp = tmp_path / "run.cfg"
    cfgp.write_text("primitive = sphere\nsubdivisions = 3\ndiameter = 0.25\nN_x = 32\nL_max = 2\n"
                    "iters_total = 8\nsample_start = 2\nsample_stride = 2\nu_in = 0.04\nRe = 10\n"
                    f"out = {tmp_path}\n")
    rc = cli.main(["simulate", "--config", str(cfgp)])
    assert rc == 0
    rows = open(tmp_path / "forces.csv").read().strip().splitlines()
    assert rows[0] == "coarse_step,F_x,F_y,F_z" and len(rows) == 1 + 3
    fx = [float(r.split(",")[1]) for r in rows[1:]]
    assert all(np.isfinite(fx)) and fx[-1] > 0  # drag along the inflow
