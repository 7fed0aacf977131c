"""GPU LUT consumer (csrc/vf_lbm.cu) against the LBM oracle
(oracle/lbm_oracle.c): one and several D3Q27 BGK collide/stream steps of the
finest level of an embedded sphere with IBB walls from the GPU's own LUT,
inlet/outlet faces, and the wall momentum exchange.
Tolerance: the GPU computes in FP32 (state stored in FP32), the oracle in
FP64 from the same FP32 state: |dF| <= 2e-6 + 2e-5 |f| per population."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from lbm_cases import perturbed_state  # noqa: E402
from paper_2512_01251_b200 import EmbedConfig, make_icosphere  # noqa: E402
from paper_2512_01251_b200.lattice import D3Q27  # noqa: E402
from paper_2512_01251_b200.solver import FlowConfig, LbmLevel  # noqa: E402
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


def _host(grid, table):
    g = grid.to_numpy()
    cmap = np.full(grid.capacity, -1, np.int32)
    cm = table.contraction_map.cpu().numpy()
    cmap[:len(cm)] = cm
    return g, cmap, table.lengths.cpu().numpy()


def _oracle_steps(O, g, cmap, lut, s, e, cells_x, f, steps, flow, ibb=True):
    force = np.zeros(3)
    for _ in range(steps):
        f, fr = O.lbm_step(g["coords"], g["nbr"], g["masks"], s, e, cells_x, cmap, lut, f, flow.tau,
                           (flow.u_in, 0.0, 0.0), ibb, flow.open_x)
        force += fr
    return f, force


@pytest.mark.parametrize("steps", [1, 3])
@pytest.mark.parametrize("scheme", ["IBB", "SBB"])
def test_step_matches_oracle(O, emb, steps, scheme):
    cfg, grid, table = emb
    L = grid.n_levels - 1
    flow = FlowConfig(Re=20.0, u_in=0.04, D_s=16.0, bc_scheme=scheme)
    lv = LbmLevel(grid, L, table, flow)
    g, cmap, lut = _host(grid, table)
    f0 = perturbed_state(g["masks"], lv.s, lv.e, np.random.default_rng(7), u=(0.04, 0, 0))
    lv.state.copy_(torch.from_numpy(f0))
    force = lv.step(steps).cpu().numpy()
    fg = lv.state.cpu().numpy()
    fo, force_o = _oracle_steps(O, g, cmap, lut, lv.s, lv.e, 4 * (cfg.nb[0] << L), f0, steps, flow,
                                ibb=scheme == "IBB")
    err = np.abs(fg - fo) - (ATOL + RTOL * np.abs(fo))
    assert err.max() <= 0, f"max excess {err.max():.3g}"
    assert np.allclose(force, force_o, rtol=1e-4, atol=1e-6 * np.abs(force_o).max())
    assert np.abs(force_o).max() > 0  # wall links were exercised


def test_ibb_half_equals_sbb(emb):
    cfg, grid, table = emb
    L = grid.n_levels - 1
    g = grid.to_numpy()
    half = table.lengths.clone()
    half[half >= 0] = 0.5
    from paper_2512_01251_b200.datatypes import LinkTable
    t_half = LinkTable(half, table.bc_ids, table.contraction_map, table.n_b)
    out = []
    for tab, scheme in ((t_half, "IBB"), (table, "SBB")):
        lv = LbmLevel(grid, L, tab, FlowConfig(u_in=0.03, D_s=16.0, bc_scheme=scheme))
        f0 = perturbed_state(g["masks"], lv.s, lv.e, np.random.default_rng(3), u=(0.03, 0, 0))
        lv.state.copy_(torch.from_numpy(f0))
        fr = lv.step(2).cpu().numpy()
        out.append((lv.state.cpu().numpy(), fr))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])


def test_rest_state_fixed_point(emb):
    cfg, grid, table = emb
    L = grid.n_levels - 1
    lv = LbmLevel(grid, L, table, FlowConfig(u_in=0.0, Re=1.0, D_s=8.0), tau=0.8)
    lv.init_equilibrium(1.0, (0.0, 0.0, 0.0))
    f0 = lv.state.clone()
    lv.step(5)
    assert (lv.state - f0).abs().max().item() < 1e-6


def test_closed_box_mass_conservation():
    mesh = make_icosphere((0.5, 0.5, 0.5), 0.4, 3)
    cfg = EmbedConfig(n_x=32, l_max=1)  # one level: no ghost layer
    grid, table = EmbedEngine(mesh, cfg, use_graph=False).run()
    lv = LbmLevel(grid, 0, table, FlowConfig(u_in=0.02, D_s=8.0, bc_scheme="SBB", open_x=False))
    g = grid.to_numpy()
    f0 = perturbed_state(g["masks"], lv.s, lv.e, np.random.default_rng(5), u=(0.02, 0.01, 0))
    lv.state.copy_(torch.from_numpy(f0))
    fluid = torch.from_numpy(g["masks"].reshape(-1)[64 * lv.s:64 * lv.e] != 1).cuda()
    m0 = lv.state[:, fluid].double().sum().item()
    lv.step(10)
    m1 = lv.state[:, fluid].double().sum().item()
    assert abs(m1 - m0) / m0 < 2e-6


def test_force_deterministic(emb):
    """the wall force is summed per block in block order, so the
    force series is bitwise identical across runs."""
    cfg, grid, table = emb
    L = grid.n_levels - 1
    g = grid.to_numpy()
    f0 = perturbed_state(g["masks"], *grid.level_range(L), np.random.default_rng(11), u=(0.04, 0, 0))
    series = []
    for _ in range(3):
        lv = LbmLevel(grid, L, table, FlowConfig(Re=20.0, u_in=0.04, D_s=16.0, bc_scheme="IBB"))
        lv.state.copy_(torch.from_numpy(f0))
        series.append(np.stack([lv.step(1).cpu().numpy().copy() for _ in range(4)]))
    assert np.abs(series[0]).max() > 0
    assert np.array_equal(series[0], series[1]) and np.array_equal(series[0], series[2])
