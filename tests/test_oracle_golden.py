"""CPU: pin the oracle (numpy + C restatements of the reference) against the
golden fixtures produced by running the reference itself (tests/golden/make_golden.py).

This is what makes the GPU parity tests meaningful: the C restatement used
as the checker at sizes numpy is too slow for is proven bitwise identical to
the reference here first."""

import math

import numpy as np
import pytest

from conftest import load_golden, sha, spacing_of

from oracle import native as ON
from oracle import waveholtz_oracle as O

SMALL = ["d1_n16", "d1_n16_p2", "d1_n4_min", "d1_n37_c13", "d2_sq32", "d2_rect", "d2_rect_p2", "d2_min",
         "d2_ragged", "d2_wide", "d2_zero", "d3_cube", "d3_box", "d3_min", "d3_ragged", "d3_thin"]


def small_case(key):
    meta, A = load_golden("small")
    case = meta["cases"][key]
    sp = spacing_of(case)
    n_t, dt, we = O.correct_explicit(case["omega"], sp, 2, case["c"], case["courant"])
    assert (n_t, dt, we) == (case["corr"]["steps_per_period"], case["corr"]["dt"], case["corr"]["omega_tilde"])
    assert O.alpha_d(we * dt) == case["corr"]["alpha"]
    return case, A, sp, O.step_scalars(n_t, dt, we, case["periods"])


@pytest.mark.parametrize("key", SMALL)
def test_numpy_oracle_bitwise(key):
    case, A, sp, sc = small_case(key)
    out = O.wave_solve_filtered(A[key + "__v"], A[key + "__f"], sp, sc, case["c"])
    assert sha(out) == case["out_sha256"]
    assert sha(O.apply_A(A[key + "__v"], sp, sc, case["c"])) == case["av_sha256"]


@pytest.mark.parametrize("key", SMALL)
def test_c_oracle_bitwise(key):
    case, A, sp, sc = small_case(key)
    out = ON.wave_solve(A[key + "__v"], A[key + "__f"], sp, sc, case["c"])
    assert sha(out) == case["out_sha256"]
    w0 = ON.wave_solve(A[key + "__v"], None, sp, sc, case["c"], zero_f=True)
    assert sha(A[key + "__v"] - w0) == case["av_sha256"]


def test_cfg1_all_100_iterates_bitwise():
    meta, A = load_golden("cfg1")
    sp = (1.0 / 128, 1.0 / 128)
    n_t, dt, we = O.correct_explicit(20.3, sp, 2, 1.0, 0.9)
    assert n_t == meta["corr"]["steps_per_period"] == 63
    sc = O.step_scalars(n_t, dt, we)
    f = O.gaussian((129, 129), [(0.0, 1.0)] * 2, sp, 100.0, 200.0, (0.4, 0.6))
    assert sha(f) == meta["f_sha256"]
    v = np.zeros_like(f)
    for k in range(3):  # numpy restatement, the exact reference ufunc sequence
        vn = O.wave_solve_filtered(v, f, sp, sc)
        r = np.linalg.norm(vn - v) / math.sqrt(v.size)
        assert sha(vn) == meta["iter_sha256"][k]
        assert abs(r - meta["residuals"][k]) <= 1e-13 * meta["residuals"][k]
        v = vn
    vc, rc = ON.fpi(f, sp, sc, 100)  # C restatement, all 100
    assert sha(vc) == meta["iter_sha256"][-1]
    assert np.array_equal(vc, A["v100"])
    np.testing.assert_allclose(rc, meta["residuals"], rtol=1e-12)


def test_cfg1_gmres_oracle():
    """The GMRES port (linalg.py:102-183) reproduces the reference's krylov_solve run."""
    meta, A = load_golden("cfg1")
    gm = meta["gmres"]
    sp = (1.0 / 128, 1.0 / 128)
    n_t, dt, we = O.correct_explicit(20.3, sp, 2, 1.0, 0.9)
    sc = O.step_scalars(n_t, dt, we)
    f = A["f"]
    b = ON.wave_solve(np.zeros_like(f), f, sp, sc)
    scale = math.sqrt(f.size)

    def matvec(x):
        return x - ON.wave_solve(x, None, sp, sc, zero_f=True)

    x, hist, iters, conv = O.gmres(matvec, b, tol=0.0, atol=gm["tol"] * scale, restart=gm["restart"],
                                   maxit=gm["maxit"])
    assert iters == gm["iterations"] and conv == gm["converged"]
    np.testing.assert_allclose([h / scale for h in hist], gm["residuals"], rtol=1e-9)
    assert np.max(np.abs(x - A["gmres_x"])) <= 1e-10 * np.max(np.abs(A["gmres_x"]))


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_large_config_first_iterate_bitwise(name):
    """First FPI iterate of configs 2 (2049^2) and 3 (257^3) through the C restatement."""
    meta, _ = load_golden(name)
    dim = meta["dim"]
    n = meta["cells"][0]
    shape = (n + 1,) * dim
    sp = (1.0 / n,) * dim
    n_t, dt, we = O.correct_explicit(meta["omega"], sp, 2, 1.0, 0.9)
    assert n_t == meta["corr"]["steps_per_period"] and dt == meta["corr"]["dt"]
    if meta["forcing"][0] == "single":
        f = O.gaussian(shape, [(0.0, 1.0)] * dim, sp, meta["forcing"][1], meta["forcing"][2], meta["forcing"][3])
    else:
        f = O.multi_gaussian(shape, [(0.0, 1.0)] * dim, sp, meta["forcing"][1], seed=0)
    assert sha(f) == meta["f_sha256"]
    sc = O.step_scalars(n_t, dt, we)
    v1 = ON.wave_solve(np.zeros(shape), f, sp, sc)
    assert sha(v1) == meta["iter_sha256"][0]
    idx = np.array(meta["sample_idx"])
    np.testing.assert_array_equal(v1.ravel()[idx], np.array(meta["samples"][0]))


def test_cfg5_schedules_and_two_frequencies():
    meta, _ = load_golden("cfg5")
    sp = (1.0 / 1024, 1.0 / 1024)
    omegas = np.linspace(10.3, 200.3, 64)
    assert np.array_equal(omegas, np.array(meta["omegas"]))
    nts = [O.correct_explicit(w, sp, 2, 1.0, 0.9)[0] for w in omegas]
    assert nts == [p["corr"]["steps_per_period"] for p in meta["per_omega"]]
    assert sum(nts) == 10522 and nts[0] == 982 and nts[-1] == 51
    f = O.multi_gaussian((1025, 1025), [(0.0, 1.0)] * 2, sp, 4, seed=0)
    assert sha(f) == meta["per_omega"][0]["f_sha256"]
    for j in (63, 40):
        n_t, dt, we = O.correct_explicit(omegas[j], sp, 2, 1.0, 0.9)
        v1 = ON.wave_solve(np.zeros((1025, 1025)), f, sp, O.step_scalars(n_t, dt, we))
        assert sha(v1) == meta["per_omega"][j]["iter_sha256"][0]


@pytest.mark.parametrize("cells,ks", [((16,), (3,)), ((20, 28), (2, 5)), ((10, 12, 14), (1, 2, 3))])
def test_eigen_action_kat_on_oracle(cells, ks):
    """W(phi, 0) = beta_d(lambda_e) phi (test_timestep.py:220-236) on the restatement."""
    sp = tuple(1.0 / n for n in cells)
    phi = O.sine_mode(cells, (1.0,) * len(cells), ks)
    lam = O.sine_mode_lambda(cells, sp, ks)
    omega = 0.8 * lam + 0.7
    n_t, dt, we = O.correct_explicit(omega, sp, 2, 1.0, 0.9)
    for periods in (1, 2):
        sc = O.step_scalars(n_t, dt, we, periods)
        out = O.wave_solve_filtered(phi, np.zeros_like(phi), sp, sc)
        beta = O.eigen_action_factor(cells, sp, ks, omega, n_t, dt, we, periods)
        assert np.max(np.abs(out - beta * phi)) <= 1e-10


EXT = ["p4_d1", "p4_d2", "p4_d2_np2", "p4_d3", "p4_min", "per_p2_d1", "per_p2_d2", "per_p2_d3", "per_p4_d1",
       "per_p4_d2", "per_p4_d3", "mix_p2_d2", "mix_p4_d2", "mix_p2_d3", "mix_p4_d3"]


@pytest.mark.parametrize("key", EXT)
def test_numpy_oracle_order4_periodic_bitwise(key):
    """order-4 stencils, periodic and mixed boundaries."""
    meta, A = load_golden("ext")
    case = meta["cases"][key]
    bcs = case["bcs"]
    sp = tuple((hi - lo) / n for (lo, hi), n in zip(case["bounds"], case["cells"]))
    p = case["order"]
    n_t, dt, we = O.correct_explicit(case["omega"], sp, p, case["c"])
    assert (n_t, dt, we) == (case["corr"]["steps_per_period"], case["corr"]["dt"], case["corr"]["omega_tilde"])
    sc = O.step_scalars(n_t, dt, we, case["periods"])
    v, f = A[key + "__v"], A[key + "__f"]
    assert sha(O.wave_solve_filtered(v, f, sp, sc, case["c"], bcs, p)) == case["out_sha256"]
    assert sha(O.apply_A(v, sp, sc, case["c"], bcs, p)) == case["av_sha256"]
    assert sha(O.laplacian_general(v, sp, bcs, p, case["c"])) == case["lap_sha256"]
