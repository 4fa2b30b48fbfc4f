"""GPU: implicit (trapezoidal) WaveHoltz on the device — SURVEY §8(f) rank 4 —
against golden outputs of the reference itself (tests/golden/implicit.*,
made by tests/golden/make_golden_implicit.py).

The inner solves are CG to 1e-12 relative (the reference's tolerance) with
device reductions instead of BLAS, so iterates are compared with the
north-star tolerance: relative max-norm error <= 1e-10 per iterate.  The
1D p = 2 case is a direct tridiagonal elimination in the reference's exact
operation order and is required to be bitwise."""

import json
import math
import os

import numpy as np
import pytest

import paper_2504_03074_b200 as wh
from paper_2504_03074_b200 import _native
from paper_2504_03074_b200.device import device_problem
from paper_2504_03074_b200.implicit import implicit_solver_for

from conftest import ROOT

pytestmark = pytest.mark.gpu

GOLD = os.path.join(ROOT, "tests", "golden")
META = json.load(open(os.path.join(GOLD, "implicit.json")))
ARR = np.load(os.path.join(GOLD, "implicit.npz"))
TOL = 1e-10


def relerr(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def setup(name):
    m = META[name]
    d = m["dim"]
    g = wh.build_grid(d, [(0.0, 1.0)] * d, m["cells"], m["bcs"])
    corr = wh.correct_implicit(m["omega"], m["n_t"])
    cfg = wh.FilterConfig(omega=m["omega"], periods=1, steps_per_period=m["n_t"], mode="implicit")
    op = wh.DiscreteOperator(g, m["order"], 1.0)
    return m, g, corr, cfg, op


@pytest.mark.parametrize("name", sorted(META))
def test_implicit_wave_solve_matches_reference(gpu_available, name):
    m, g, corr, cfg, op = setup(name)
    f = wh.GridField.from_values(g, ARR[f"{name}/f"])
    v0 = wh.GridField.from_values(g, ARR[f"{name}/v0"])

    class Counter:
        inner = 0

    cnt = Counter()
    out = wh.wave_solve_filtered(v0, f, cfg, corr, op, linear_solver=cnt,
                                 implicit_first_step=m["implicit_first_step"]).values
    ref = ARR[f"{name}/out"]
    if name == "tri1d_p2":
        assert np.array_equal(out, ref)
    else:
        assert relerr(out, ref) <= TOL, relerr(out, ref)
    # same solver family, same amount of inner work (CG counts may differ by a step at the tolerance edge)
    assert abs(cnt.inner - m["inner"]) <= max(2, 0.03 * m["inner"]), (cnt.inner, m["inner"])
    s = implicit_solver_for(device_problem(g, 1.0, m["order"]), g, m["order"], 1.0, corr.dt)
    assert s.precond == (m["precond"] if m["order"] == 4 or m["precond"] != "tri" else None) or s.direct


@pytest.mark.parametrize("name", [n for n in sorted(META) if "fpi_residuals" in META[n]])
def test_implicit_fpi_iterates(gpu_available, name):
    m, g, corr, cfg, op = setup(name)
    prob = wh.HelmholtzProblem(g, m["order"], 1.0, m["omega"], wh.GridField.from_values(g, ARR[f"{name}/f"]))
    k = len(m["fpi_residuals"])
    v, run = wh.fpi_solve(prob, cfg, tol=-1.0, maxit=k)
    ref = ARR[f"{name}/fpi{k}"]
    assert relerr(v.values, ref) <= TOL
    np.testing.assert_allclose(run.residuals, m["fpi_residuals"], rtol=1e-9)
    assert run.inner_iterations > 0


def test_implicit_gmres(gpu_available):
    name = "gmres2d"
    m, g, corr, cfg, op = setup(name)
    prob = wh.HelmholtzProblem(g, m["order"], 1.0, m["omega"], wh.GridField.from_values(g, ARR[f"{name}/f"]))
    x, run = wh.krylov_solve(prob, cfg, tol=m["gmres"]["tol"], restart=m["gmres"]["restart"])
    assert run.iterations == m["gmres"]["iterations"]
    assert relerr(x.values, ARR[f"{name}/gmres_x"]) <= 1e-8  # GMRES stops at 1e-9: solutions agree to that
    np.testing.assert_allclose(run.residuals, m["gmres"]["residuals"], rtol=1e-6)


def test_implicit_cg_residual_at_scale(gpu_available):
    """Size-independent property at 1025^2 (no CPU reference needed): every implicit solve
    meets ||rhs - A w|| <= 1e-12 ||rhs||, checked on the device for one step."""
    g = wh.build_grid(2, [(0.0, 1.0)] * 2, (1024, 1024), "dirichlet")
    corr = wh.correct_implicit(60.0, 10)
    dp = device_problem(g)
    s = implicit_solver_for(dp, g, 2, 1.0, corr.dt)
    assert s.precond == "mg"
    ctx = dp.ctx
    rhs, x, ax = ctx.vec_reserve(3)
    rng = np.random.default_rng(0)
    ctx.vec_upload(rhs, rng.standard_normal(g.shape))
    its = s.solve(rhs, rhs, x)
    s.apply(x, ax)
    ctx.sub_into(rhs, ax, ax)
    rel = math.sqrt(ctx.dot(ax, ax)) / math.sqrt(ctx.dot(rhs, rhs))
    assert rel <= 1.5e-12 and 0 < its < 60, (rel, its)


@pytest.mark.parametrize("dim,cells,bcs,order,omega,n_t", [(2, (256, 256), "dirichlet", 2, 30.0, 10),
                                                          (2, (128, 192), "dirichlet", 4, 25.0, 8),
                                                          (1, (4096,), "dirichlet", 2, 40.0, 12),
                                                          (3, (24, 20, 28), "dirichlet", 2, 9.0, 6),
                                                          (2, (60, 50), "periodic", 2, 12.0, 7)])
def test_implicit_against_oracle_larger(gpu_available, dim, cells, bcs, order, omega, n_t):
    """Beyond the fixture sizes: the device against the oracle restatement (pinned bitwise to
    the reference by tests/test_oracle_implicit.py)."""
    from oracle import implicit_oracle as IO
    from oracle import waveholtz_oracle as O

    g = wh.build_grid(dim, [(0.0, 1.0)] * dim, cells, bcs)
    f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=4)
    if bcs == "periodic":
        f = np.array(f)
    v0 = O.zero_dirichlet(np.random.default_rng(9).standard_normal(g.shape) * 1e-2, [bcs] * dim)
    corr = wh.correct_implicit(omega, n_t)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=n_t, mode="implicit")
    op = wh.DiscreteOperator(g, order, 1.0)
    out = wh.wave_solve_filtered(wh.GridField.from_values(g, v0), wh.GridField.from_values(g, f), cfg, corr,
                                 op).values
    ref, solver = IO.wave_solve_implicit(v0, np.array(wh.GridField.from_values(g, f).values), g.spacing,
                                         [bcs] * dim, order, omega, n_t)
    assert relerr(out, ref) <= TOL, relerr(out, ref)


@pytest.mark.parametrize("cells", [(256, 256), (512, 128), (128, 64), (1024, 1024), (192, 320)])
def test_vcycle_single_cta_coarse_path_bitwise(gpu_available, monkeypatch, cells):
    """The single-CTA coarse sub-cycle (shared memory) and the temporally blocked smoother (four
    half-sweeps per launch) compute exactly what the per-level / per-colour kernels compute:
    one V-cycle both ways, bitwise."""
    from paper_2504_03074_b200.device import DeviceProblem
    from paper_2504_03074_b200.implicit import DeviceImplicitSolver

    g = wh.build_grid(2, [(0.0, 1.0)] * 2, cells, "dirichlet")
    dt = wh.correct_implicit(20.0, 10).dt
    r = np.random.default_rng(5).standard_normal(g.shape)
    outs = []
    for env in ("1", "0"):
        monkeypatch.setenv("WHB_MG_COARSE_CTA", env)
        monkeypatch.setenv("WHB_GS_BLOCK", env)
        dp = DeviceProblem(g)
        s = DeviceImplicitSolver(dp.ctx, g, 2, 1.0, dt)
        dp.ctx.vec_upload(s.r, r)
        dp.ctx.mg_vcycle(s.r, s.z)
        outs.append(dp.ctx.vec_download(s.z))
        dp.close()
    assert np.array_equal(outs[0], outs[1])
    assert np.any(outs[0] != 0.0)


def test_mixed_explicit_implicit_calls_share_one_device_problem(gpu_available):
    """Explicit and implicit solves, FPI, GMRES and single wave solves interleaved on one cached
    device problem (shared fields, vectors and graphs): every result matches its checker."""
    from oracle import implicit_oracle as IO
    from oracle import native as ON
    from oracle import waveholtz_oracle as O

    g = wh.build_grid(2, [(0.0, 1.0)] * 2, (64, 64), "dirichlet")
    f = wh.multi_gaussian_source(g, 9.0, 3, seed=8)
    fv = np.array(f.values)
    op = wh.DiscreteOperator(g, 2, 1.0)
    for rnd in range(2):
        for omega in (7.5, 10.0):
            prob = wh.HelmholtzProblem(g, 2, 1.0, omega, f)
            # explicit FPI (bitwise)
            cfg_e = wh.FilterConfig(omega=omega, mode="explicit")
            v, run = wh.fpi_solve(prob, cfg_e, tol=-1.0, maxit=2)
            corr_e = wh.correct_explicit(omega, g, 2, 1.0)
            sc = O.step_scalars(corr_e.steps_per_period, corr_e.dt, corr_e.omega_tilde)
            vref, rref = ON.fpi(fv, g.spacing, sc, 2)
            assert np.array_equal(v.values, vref)
            np.testing.assert_allclose(run.residuals, rref, rtol=1e-12)
            # implicit single solve from that iterate (<= 1e-10)
            cfg_i = wh.FilterConfig(omega=omega, periods=1, steps_per_period=8, mode="implicit")
            corr_i = wh.correct_implicit(omega, 8)
            out = wh.wave_solve_filtered(v, f, cfg_i, corr_i, op).values
            ref, _ = IO.wave_solve_implicit(np.array(v.values), fv, g.spacing, ["dirichlet"] * 2, 2, omega, 8)
            assert relerr(out, ref) <= TOL
            # explicit single solve again (bitwise)
            out_e = wh.wave_solve_filtered(v, f, cfg_e.__class__(omega=omega, periods=1,
                                                                  steps_per_period=corr_e.steps_per_period,
                                                                  mode="explicit"), corr_e, op).values
            assert np.array_equal(out_e, ON.wave_solve(np.array(v.values), fv, g.spacing, sc))
            # implicit FPI
            vi, runi = wh.fpi_solve(prob, cfg_i, tol=-1.0, maxit=2)
            w = np.zeros_like(fv)
            solver = None
            for _ in range(2):
                w, solver = IO.wave_solve_implicit(w, fv, g.spacing, ["dirichlet"] * 2, 2, omega, 8, solver=solver)
            assert relerr(vi.values, w) <= TOL


def test_host_fpi_step_implicit(gpu_available):
    """HostFPIStep (host buffers in and out each pass) in implicit mode reproduces fpi_solve's
    device-resident iterates and residuals."""
    name = "mg2d_64"
    m, g, corr, cfg, op = setup(name)
    prob = wh.HelmholtzProblem(g, m["order"], 1.0, m["omega"], wh.GridField.from_values(g, ARR[f"{name}/f"]))
    step = wh.HostFPIStep(prob, cfg)
    a, b = np.zeros(g.shape), np.zeros(g.shape)
    res = []
    for _ in range(3):
        res.append(step(a, b))
        a, b = b, a
    v, run = wh.fpi_solve(prob, cfg, tol=-1.0, maxit=3)
    assert np.array_equal(a, v.values)
    np.testing.assert_allclose(res, run.residuals, rtol=1e-13)
    assert relerr(a, ARR[f"{name}/fpi3"]) <= TOL


@pytest.mark.parametrize("dim,cells,order", [(1, (300,), 2), (1, (256,), 4), (2, (64, 64), 2)])
def test_solvers_of_different_dt_interleaved_on_one_grid(gpu_available, dim, cells, order):
    """One context holds one tridiagonal factorisation / multigrid hierarchy.  Solvers for
    omegas A, B, A (different dt) held at the same time and used in that order must each run
    on their own factors (the cached solver A used to run against B's state; in 2D
    its CG graph replayed kernels pointing at freed multigrid buffers)."""
    from oracle import implicit_oracle as IO
    from oracle import waveholtz_oracle as O

    g = wh.build_grid(dim, [(0.0, 1.0)] * dim, cells, "dirichlet")
    f = np.array(O.multi_gaussian(g.shape, g.bounds, g.spacing, 2, seed=3))
    v0 = O.zero_dirichlet(np.random.default_rng(2).standard_normal(g.shape) * 1e-2, ["dirichlet"] * dim)
    op = wh.DiscreteOperator(g, order, 1.0)
    dp = device_problem(g, order=order)
    outs = {}
    for omega in (12.0, 21.0, 12.0, 21.0):
        n_t = 9
        corr = wh.correct_implicit(omega, n_t)
        cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=n_t, mode="implicit")
        # hold both solvers: the second call of each omega reuses its cached solver
        implicit_solver_for(dp, g, order, 1.0, wh.correct_implicit(12.0, n_t).dt)
        implicit_solver_for(dp, g, order, 1.0, wh.correct_implicit(21.0, n_t).dt)
        out = wh.wave_solve_filtered(wh.GridField.from_values(g, v0), wh.GridField.from_values(g, f), cfg, corr,
                                     op).values
        ref, _ = IO.wave_solve_implicit(v0, np.array(wh.GridField.from_values(g, f).values), g.spacing,
                                        ["dirichlet"] * dim, order, omega, n_t)
        tol = 0.0 if (dim == 1 and order == 2) else TOL  # 1D p = 2: direct elimination, bitwise
        assert relerr(out, ref) <= tol, (omega, relerr(out, ref))
        if omega in outs:
            assert np.array_equal(outs[omega], out)
        outs[omega] = out
