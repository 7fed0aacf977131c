"""CPU checks of the LBM oracle (oracle/lbm_oracle.c), the checker of the
GPU collide/stream kernel: equilibrium moments, the rest
state as a fixed point of every boundary rule, IBB at q = 1/2 equal to SBB
(SPEC.md:410), and mass conservation in a closed SBB box."""
import numpy as np
import pytest

from lbm_cases import level_arrays, perturbed_state, sphere_case
from paper_2512_01251_b200.lattice import D3Q27
from paper_2512_01251_b200.solver import FlowConfig, equilibrium


@pytest.fixture(scope="module")
def O(oracle_mod):
    return oracle_mod


@pytest.fixture(scope="module")
def case(O):
    return sphere_case(O)


def test_equilibrium_moments(O):
    rng = np.random.default_rng(0)
    for _ in range(20):
        rho = 0.8 + 0.4 * rng.random()
        u = 0.1 * (rng.random(3) - 0.5)
        f = O.lbm_equilibrium(rho, u)
        assert np.allclose(f, equilibrium(rho, u), rtol=1e-14, atol=0)
        assert abs(f.sum() - rho) < 1e-14
        assert np.allclose(f @ D3Q27.c, rho * u, atol=1e-15)
    assert np.allclose(O.lbm_equilibrium(1.0, [0, 0, 0]), D3Q27.w, rtol=0, atol=1e-16)


def test_flow_tau():
    assert abs(FlowConfig(Re=20, u_in=0.05, D_s=8).tau - (0.05 * 8 / 20 * 3 + 0.5)) < 1e-15
    with pytest.raises(ValueError):
        _ = FlowConfig(Re=20, u_in=0.0, D_s=8).tau


def _step(O, ref, cfg, L, f, ibb=True, open_x=True, u_in=(0.0, 0.0, 0.0), tau=0.6, lengths=None):
    g, s, e = level_arrays(ref, L)
    cmap = np.full(g.capacity, -1, np.int32)
    cmap[:len(ref.contraction_map)] = ref.contraction_map
    lut = ref.lengths if lengths is None else lengths
    return O.lbm_step(g.coords, g.nbr, g.masks, s, e, 4 * (cfg.nb[0] << L), cmap,
                      lut if len(lut) else np.zeros((1, 27, 64), np.float32), f, tau, u_in, ibb, open_x)


def test_rest_state_fixed_point(O, case):
    _, cfg, ref = case
    L = cfg.l_max - 1
    g, s, e = level_arrays(ref, L)
    n = (e - s) * 64
    f = np.repeat(D3Q27.w[:, None], n, axis=1).astype(np.float32)
    f[:, g.masks.reshape(-1)[64 * s:64 * e] == 1] = 0.0
    for ibb in (True, False):
        out, force = _step(O, ref, cfg, L, f, ibb=ibb)
        assert np.abs(out - f).max() < 1e-7
        assert np.abs(force).max() < 1e-12 * max(1.0, np.abs(force).sum())


def test_ibb_half_equals_sbb(O, case):
    _, cfg, ref = case
    L = cfg.l_max - 1
    g, s, e = level_arrays(ref, L)
    f = perturbed_state(g.masks, s, e, np.random.default_rng(1))
    half = np.where(ref.lengths >= 0, np.float32(0.5), ref.lengths).astype(np.float32)
    a, fa = _step(O, ref, cfg, L, f, ibb=True, lengths=half, u_in=(0.03, 0, 0))
    b, fb = _step(O, ref, cfg, L, f, ibb=False, u_in=(0.03, 0, 0))
    assert np.array_equal(a, b)
    assert np.array_equal(fa, fb)


def test_closed_box_mass_conservation(O):
    # one level (no ghost layer): SBB walls and box faces conserve mass exactly
    _, cfg, ref = sphere_case(O, l_max=1, n_x=32)
    g, s, e = level_arrays(ref, 0)
    f = perturbed_state(g.masks, s, e, np.random.default_rng(2), u=(0.02, 0.01, 0.0))
    fluid = g.masks.reshape(-1)[64 * s:64 * e] != 1
    m0 = f[:, fluid].astype(np.float64).sum()
    for _ in range(3):
        f, _ = _step(O, ref, cfg, 0, f, ibb=False, open_x=False)
    m1 = f[:, fluid].astype(np.float64).sum()
    assert abs(m1 - m0) / m0 < 1e-6
