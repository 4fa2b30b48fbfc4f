"""CPU: the host-side mirror of the reference interface (no GPU needed).

Scalars handed to the kernels must be bitwise what the reference computes
(time correction, per-step schedule, stencil coefficients, forcing), and the
Python surface must raise the reference's exception types."""

import contextlib
import math

import numpy as np
import pytest

from conftest import load_golden, sha

import paper_2504_03074_b200 as wh
from paper_2504_03074_b200 import grid as G
from paper_2504_03074_b200 import timestep as ts
from oracle import reference_harness as RH
from oracle import waveholtz_oracle as O


@contextlib.contextmanager
def courant(value):
    old = ts._COURANT[2]
    ts._COURANT[2] = value
    try:
        yield
    finally:
        ts._COURANT[2] = old


@pytest.mark.parametrize("omega,n,dim,nt", [(20.3, 128, 2, 63), (100.5, 2048, 2, 202), (40.7, 256, 3, 77),
                                            (150.3, 1024, 3, 83), (200.3, 1024, 2, 51), (10.3, 1024, 2, 982)])
def test_correct_explicit_cfl09_appendix_b(omega, n, dim, nt):
    g = wh.build_grid(dim, [(0.0, 1.0)] * dim, [n] * dim, "dirichlet")
    with courant(0.9):
        corr = wh.correct_explicit(omega, g, 2, 1.0)
    assert corr.steps_per_period == nt
    assert (corr.steps_per_period, corr.dt, corr.omega_tilde) == O.correct_explicit(omega, g.spacing, 2, 1.0, 0.9)
    assert abs(math.sin(corr.omega_tilde * corr.dt / 2) / (corr.dt / 2) - omega) <= 1e-13 * omega


def test_reference_default_courant_counts():
    """Unpatched Courant bound 1.0 gives 57 / 182 / 69 / 75."""
    for omega, n, dim, nt in [(20.3, 128, 2, 57), (100.5, 2048, 2, 182), (40.7, 256, 3, 69), (150.3, 1024, 3, 75)]:
        g = wh.build_grid(dim, [(0.0, 1.0)] * dim, [n] * dim, "dirichlet")
        assert wh.correct_explicit(omega, g, 2, 1.0).steps_per_period == nt


@pytest.mark.parametrize("periods", [1, 2, 3])
def test_time_schedule_bitwise_vs_oracle(periods):
    g = wh.build_grid(2, [(0.0, 1.0), (0.0, 2.0)], [24, 40], "dirichlet")
    corr = wh.correct_explicit(7.1, g, 2, 1.3)
    cfg = wh.FilterConfig(omega=7.1, periods=periods, steps_per_period=corr.steps_per_period, mode="explicit")
    s = wh.time_schedule(corr, cfg)
    o = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde, periods)
    assert s["n_total"] == o["n_total"] == periods * corr.steps_per_period
    for k in ("half_dt2", "dt2", "out_scale"):
        assert s[k] == o[k]
    assert np.array_equal(s["cos_f"][1:], o["cos_f"][1:])
    assert np.array_equal(s["acc_c"], o["acc_c"])
    assert corr.alpha == o["alpha"]


def test_operator_coefficients_match_reference_taps():
    g = wh.build_grid(3, [(0.0, 1.0), (0.0, 0.8), (-0.5, 1.0)], [12, 10, 14], "dirichlet")
    clo, cmid, c2 = G.operator_coefficients(g, 2, 0.8)
    for a, dx in enumerate(g.spacing):
        taps = np.array([1.0, -2.0, 1.0]) / dx**2
        assert clo[a] == taps[0] and cmid[a] == taps[1]
    assert c2 == 0.8**2
    with pytest.raises(NotImplementedError):
        G.operator_coefficients(g, 4, 1.0)
    gp = wh.build_grid(2, [(0.0, 1.0)] * 2, [8, 8], "periodic")
    with pytest.raises(NotImplementedError):
        G.operator_coefficients(gp, 2, 1.0)


def test_gaussian_sources_match_golden_bits():
    meta1, A1 = load_golden("cfg1")
    g = wh.build_grid(2, [(0.0, 1.0)] * 2, [128, 128], "dirichlet")
    assert sha(wh.gaussian_source(g, 20.3, 100.0, 200.0, (0.4, 0.6)).values) == meta1["f_sha256"]
    meta, _ = load_golden("small")
    _, A = load_golden("small")
    g3 = wh.build_grid(3, [(0.0, 1.0)] * 3, [16, 16, 16], "dirichlet")
    assert np.array_equal(wh.gaussian_source(g3, 9.0, 100.0, 30.0, (0.45, 0.5, 0.55)).values, A["fpi3d__f"])


def test_multi_gaussian_recipe_cfg2_cfg5():
    meta2, _ = load_golden("cfg2")
    g2 = wh.build_grid(2, [(0.0, 1.0)] * 2, [2048, 2048], "dirichlet")
    assert sha(wh.multi_gaussian_source(g2, 100.5, 8, seed=0).values) == meta2["f_sha256"]
    meta5, _ = load_golden("cfg5")
    g5 = wh.build_grid(2, [(0.0, 1.0)] * 2, [1024, 1024], "dirichlet")
    assert sha(wh.multi_gaussian_source(g5, 150.3, 4, seed=0).values) == meta5["per_omega"][0]["f_sha256"]


def test_multi_gaussian_slab_generation_is_bitwise_identical():
    g = wh.build_grid(3, [(0.0, 1.0)] * 3, [40, 33, 37], "dirichlet")
    whole = wh.multi_gaussian_source(g, 5.0, 5, seed=3).values
    for slab in (1, 7, 16):
        assert np.array_equal(wh.multi_gaussian_source(g, 5.0, 5, seed=3, slab_planes=slab).values, whole)
    assert np.array_equal(whole, O.multi_gaussian(g.shape, g.bounds, g.spacing, 5, seed=3))


def test_resonance_gap_and_error():
    g = wh.build_grid(2, [(0.0, 1.0)] * 2, [32, 32], "dirichlet")
    lam = O.sine_mode_lambda((32, 32), g.spacing, (3, 4))
    gap = wh.driver.resonance_gap(g, 2, 1.0, lam * (1 + 1e-6))
    assert gap <= 1.0000001e-6
    with pytest.raises(wh.ResonanceError):
        wh.HelmholtzProblem(g, 2, 1.0, lam, wh.GridField.zeros(g))
    # brute force over every mode
    ms = np.arange(1, 32)
    l2 = (1.0 / g.spacing[0]) ** 2 * 4 * np.sin(ms * np.pi / 64) ** 2
    full = np.sqrt(np.add.outer(l2, l2)).ravel()
    for omega in (5.7, 20.3, 91.0):
        assert abs(wh.driver.resonance_gap(g, 2, 1.0, omega) - np.min(np.abs(omega - full)) / omega) <= 1e-15


@pytest.mark.skipif(not RH.available(), reason="reference not present")
def test_resonance_gap_matches_reference_eigenvalues():
    wh_ref = RH.import_reference()
    g = wh.build_grid(2, [(0.0, 1.0), (0.0, 1.5)], [30, 44], "dirichlet")
    gr = wh_ref.grid.build_grid(2, [(0.0, 1.0), (0.0, 1.5)], [30, 44], "dirichlet")
    lam = wh_ref.grid.discrete_eigenvalues_symbolic(gr, 2, 1.3)
    for omega in (4.4, 33.3, 71.7):
        ref = np.min(np.abs(omega - lam)) / omega
        assert abs(wh.driver.resonance_gap(g, 2, 1.3, omega) - ref) <= 1e-14


def test_grid_and_config_validation():
    with pytest.raises(ValueError):
        wh.build_grid(2, (0.0, 1.0), 8, "dirichlet")
    with pytest.raises(ValueError):
        wh.build_grid(1, (0.0, 1.0), 3, "dirichlet")
    with pytest.raises(ValueError):
        wh.build_grid(2, [(0.0, 1.0)] * 2, 8, [("periodic", "dirichlet"), "dirichlet"])
    with pytest.raises(ValueError):
        wh.CartesianGrid(4, ((0, 1),) * 4, (8,) * 4, (G.BC.DIRICHLET,) * 4)
    g = wh.build_grid(3, [(0.0, 1.0)] * 3, 8, "dirichlet")
    assert g.shape == (9, 9, 9) and g.size == 729
    f = wh.GridField.from_values(g, np.ones(g.shape))
    assert f.values[0, 3, 3] == 0.0 and f.values[4, 4, 4] == 1.0 and f.generation == 1
    with pytest.raises(ValueError):
        f.values[1, 1, 1] = 2.0
    with pytest.raises(ValueError):
        wh.FilterConfig(omega=1.0, steps_per_period=4, mode="implicit")
    with pytest.raises(ValueError):
        wh.alpha_d(2.0)
    assert abs(wh.alpha_d(1e-4) - 0.5) < 1e-8


def test_mode_errors_raise_before_any_device_work():
    g = wh.build_grid(2, [(0.0, 1.0)] * 2, 16, "dirichlet")
    op = wh.DiscreteOperator(g, 2)
    corr = wh.correct_explicit(5.0, g, 2, 1.0)
    cfg_i = wh.FilterConfig(omega=5.0, periods=1, steps_per_period=10, mode="implicit")
    with pytest.raises(ValueError, match="mode"):
        wh.wave_solve_filtered(wh.GridField.zeros(g), wh.GridField.zeros(g), cfg_i, corr, op)
    prob = wh.HelmholtzProblem(g, 2, 1.0, 5.0, wh.GridField.zeros(g))
    corr_i, cfg2 = wh.resolve_time_discretization(prob, cfg_i)  # implicit: N_t from the config
    assert cfg2 is cfg_i and corr_i.steps_per_period == 10 and corr_i == wh.correct_implicit(5.0, 10)
    with pytest.raises(ValueError, match="steps per period"):
        wh.wave_solve_filtered(wh.GridField.zeros(g), wh.GridField.zeros(g), cfg_i, wh.correct_implicit(5.0, 12), op)
    with pytest.raises(ValueError):
        wh.correct_implicit(5.0, 4)
    with pytest.raises(ValueError):
        wh.resolve_time_discretization(prob, wh.FilterConfig(omega=5.0, mode="continuous"))


def test_measure_rate():
    run = wh.WaveHoltzRun("fpi", 2, [1.0, 0.5, 0.25, 0.125, 0.0625, 0.03125], 6, False)
    cr, ecr = wh.measure_rate(run)
    assert abs(cr - 0.5) < 1e-15 and abs(ecr - math.sqrt(0.5)) < 1e-15
    with pytest.raises(ValueError):
        wh.measure_rate(wh.WaveHoltzRun("fpi", 1, [1.0, 0.5], 2, False))
