"""GPU: SURVEY §8(f) rank 2 — order-4 stencils, periodic and mixed boundaries on
the device (general one-step kernel), bitwise against the reference's outputs
(tests/golden/ext.*, produced by tests/golden/make_golden.py ext)."""

import math

import numpy as np
import pytest

from conftest import load_golden, rel_maxnorm, sha

import paper_2504_03074_b200 as wh
from oracle import waveholtz_oracle as O

pytestmark = pytest.mark.gpu

EXT = ["p4_d1", "p4_d2", "p4_d2_np2", "p4_d3", "p4_min", "per_p2_d1", "per_p2_d2", "per_p2_d3", "per_p4_d1",
       "per_p4_d2", "per_p4_d3", "mix_p2_d2", "mix_p4_d2", "mix_p2_d3", "mix_p4_d3"]


def grid_of(case):
    return wh.build_grid(case["dim"], [tuple(b) for b in case["bounds"]], case["cells"], case["bcs"])


@pytest.fixture(params=["march", "grid-stride"])
def general_kernel(request, monkeypatch):
    """Both general-operator kernels: the marching one (default) and the grid-stride one
    (WHB_GEN_MARCH=0); the plan is made when a context gets the operator, so fresh contexts."""
    wh.release_device_cache()
    if request.param == "grid-stride":
        monkeypatch.setenv("WHB_GEN_MARCH", "0")
    yield request.param
    wh.release_device_cache()


@pytest.mark.parametrize("key", EXT)
def test_general_operator_wave_solve_bitwise(gpu_available, general_kernel, key):
    meta, A = load_golden("ext")
    case = meta["cases"][key]
    g = grid_of(case)
    p = case["order"]
    corr = wh.correct_explicit(case["omega"], g, p, case["c"])
    assert corr.steps_per_period == case["corr"]["steps_per_period"] and corr.dt == case["corr"]["dt"]
    cfg = wh.FilterConfig(omega=case["omega"], periods=case["periods"], steps_per_period=corr.steps_per_period,
                          mode="explicit")
    op = wh.DiscreteOperator(g, p, case["c"])
    v = wh.GridField.from_values(g, A[key + "__v"])
    f = wh.GridField.from_values(g, A[key + "__f"])
    out = wh.wave_solve_filtered(v, f, cfg, corr, op)
    assert rel_maxnorm(out.values, A[key + "__out"]) <= 1e-10
    assert sha(out.values) == case["out_sha256"]
    assert sha(op.apply_values(v.values)) == case["lap_sha256"]
    prob = type("P", (), {"grid": g, "order": p, "c": case["c"], "omega": case["omega"]})()
    assert sha(wh.waveholtz_operator(prob, cfg, corr=corr)(A[key + "__v"])) == case["av_sha256"]


def test_fpi_periodic_order4_bitwise(gpu_available, general_kernel):
    meta, A = load_golden("ext")
    case = meta["cases"]["fpi_per_p4"]
    g = wh.build_grid(2, [(0.0, 1.0)] * 2, [24, 24], "periodic")
    f = wh.gaussian_source(g, 6.1, -80.0, 25.0, (0.45, 0.55))
    assert np.array_equal(f.values, A["fpi_per_p4__f"])
    prob = wh.HelmholtzProblem(g, 4, 1.0, 6.1, f)
    cfg = wh.FilterConfig(omega=6.1, periods=1, steps_per_period=10, mode="explicit")
    dp = wh.device.device_problem(g, order=4)
    corr, cfg_e = wh.resolve_time_discretization(prob, cfg)
    dp.set_schedule(wh.time_schedule(corr, cfg_e))
    dp.set_forcing(f.values)
    from paper_2504_03074_b200 import _native

    dp.ctx.zero(_native.V)
    for k in range(5):
        r = math.sqrt(dp.ctx.fpi(1)[0, 0]) / math.sqrt(g.size)
        assert sha(dp.ctx.download(_native.V)) == case["iter_sha256"][k]
        assert abs(r - case["residuals"][k]) <= 1e-12 * case["residuals"][k]


def test_krylov_order4_matches_reference(gpu_available):
    meta, A = load_golden("ext")
    case = meta["cases"]["gmres_p4_1d"]
    g = wh.build_grid(1, (0.0, 1.0), 32, "dirichlet")
    f = wh.gaussian_source(g, 5.5, -100.0, 30.0, 0.37)
    assert np.array_equal(f.values, A["gmres_p4_1d__f"])
    prob = wh.HelmholtzProblem(g, 4, 1.0, 5.5, f)
    cfg = wh.FilterConfig(omega=5.5, periods=1, steps_per_period=10, mode="explicit")
    x, run = wh.krylov_solve(prob, cfg, tol=1e-10)
    assert run.iterations == case["iterations"]
    np.testing.assert_allclose(run.residuals, case["residuals"], rtol=1e-6)
    assert rel_maxnorm(x.values, A["gmres_p4_1d__x"]) <= 1e-9
    v, runf = wh.fpi_solve(prob, cfg, tol=1e-10, maxit=800)
    assert runf.iterations == case["fpi_iterations"]
    assert rel_maxnorm(v.values, A["gmres_p4_1d__fpi"]) <= 1e-10


@pytest.mark.parametrize("cells,bcs,p", [((160, 130), "periodic", 4), ((96, 80), ["periodic", "dirichlet"], 2),
                                         ((40, 36, 44), "dirichlet", 4), ((32, 30, 28), "periodic", 2)])
def test_general_operator_larger_grids_vs_oracle(gpu_available, cells, bcs, p):
    d = len(cells)
    g = wh.build_grid(d, [(0.0, 1.0)] * d, list(cells), bcs)
    rng = np.random.default_rng(4)
    v = wh.GridField.from_values(g, rng.standard_normal(g.shape))
    f = wh.GridField.from_values(g, rng.standard_normal(g.shape))
    corr = wh.correct_explicit(9.0, g, p, 1.0)
    cfg = wh.FilterConfig(omega=9.0, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    out = wh.wave_solve_filtered(v, f, cfg, corr, wh.DiscreteOperator(g, p, 1.0))
    names = [getattr(b, "value", b) for b in g.bcs]
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    ref = O.wave_solve_filtered(np.array(v.values), np.array(f.values), g.spacing, sc, 1.0, names, p)
    assert np.array_equal(out.values, ref)


@pytest.mark.parametrize("dim,cells,bcs,order", [(3, (40, 33, 70), "periodic", 4), (2, (300, 257), "dirichlet", 4),
                                                 (3, (24, 30, 36), ["periodic", "dirichlet", "periodic"], 2)])
def test_general_kernels_larger_grids_against_oracle(gpu_available, general_kernel, dim, cells, bcs, order):
    """Beyond the fixture sizes (several axis-0 chunks and axis-2 tiles of the marching kernel):
    one W(v, f) bitwise against the numpy restatement (oracle/waveholtz_oracle.py)."""
    g = wh.build_grid(dim, [(0.0, 1.0)] * dim, cells, bcs)
    bl = [bcs] * dim if isinstance(bcs, str) else list(bcs)
    f = np.array(O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=11))
    v = O.zero_dirichlet(np.random.default_rng(2).standard_normal(g.shape) * 1e-2, bl)
    f = O.zero_dirichlet(f, bl)
    corr = wh.correct_explicit(8.5, g, order, 1.0)
    cfg = wh.FilterConfig(omega=8.5, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    out = wh.wave_solve_filtered(wh.GridField.from_values(g, v), wh.GridField.from_values(g, f), cfg, corr,
                                 wh.DiscreteOperator(g, order, 1.0)).values
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    ref = O.wave_solve_filtered(v, f, g.spacing, sc, 1.0, bl, order)
    assert np.array_equal(out, ref)
