"""GPU: the host-callable API beside the hot path against the reference's own outputs
(tests/golden/api.*, tests/golden/make_golden_api.py): gmres_solve (linalg.py:102-183) with
device Krylov vectors, step_implicit + make_implicit_solver (timestep.py:148-247) on the device
implicit solver.  Tolerances: GMRES same iteration count, residual history to 1e-9 relative,
x to 1e-10; implicit steps north-star 1e-10 relative max-norm (1D p = 2 bitwise)."""

import json
import os

import numpy as np
import pytest

from conftest import ROOT

import paper_2504_03074_b200 as wh

pytestmark = pytest.mark.gpu
META = json.load(open(os.path.join(ROOT, "tests", "golden", "api.json")))
ARR = np.load(os.path.join(ROOT, "tests", "golden", "api.npz"))


def relerr(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("key,kw", [("dense", {}), ("dense_x0", {"x0": "x0"}), ("dense_atol", {"atol": 1e-6, "tol": 0.0})])
def test_gmres_solve_dense(gpu_available, key, kw):
    kw = {k: (ARR[v] if isinstance(v, str) else v) for k, v in kw.items()}
    x, rep = wh.gmres_solve(ARR["A"], ARR["b"], restart=12, maxit=200, **{"tol": 1e-10, **kw})
    m = META[key]
    assert rep.iterations == m["iterations"] and rep.converged == m["converged"]
    np.testing.assert_allclose(rep.residual_history, m["history"], rtol=1e-9)
    assert relerr(x, ARR[f"{key}__x"]) <= 1e-10


def test_gmres_solve_callable_on_2d_arrays(gpu_available):
    D = ARR["D"]

    def op(v):
        out = D * v
        out[1:, :] += 0.3 * v[:-1, :]
        out[:, :-1] -= 0.2 * v[:, 1:]
        return out

    seen = []
    x, rep = wh.gmres_solve(op, ARR["B"], tol=1e-11, restart=25, maxit=300, callback=seen.append)
    m = META["callable"]
    assert x.shape == ARR["B"].shape
    assert rep.iterations == m["iterations"] and len(seen) == rep.iterations
    np.testing.assert_allclose(rep.residual_history, m["history"], rtol=1e-9)
    assert relerr(x, ARR["callable__x"]) <= 1e-10


@pytest.mark.parametrize("key", ["imp1d", "imp2d", "imp1d_p4"])
def test_step_implicit_with_make_implicit_solver(gpu_available, key):
    m = META[key]
    g = wh.build_grid(m["dim"], [(0.0, 1.0)] * m["dim"], m["cells"], "dirichlet")
    op = wh.DiscreteOperator(g, m["order"], 1.0)
    corr = wh.correct_implicit(m["omega"], m["n_t"])
    solver = wh.make_implicit_solver(op, corr.dt, tol=1e-12)
    st = wh.WaveState.start(ARR[f"{key}__v0"])
    for k in range(5):
        st = wh.step_implicit(st, op, ARR[f"{key}__f"], corr, solver)
        ref = ARR[f"{key}__w"][k]
        if key == "imp1d":
            assert np.array_equal(st.w, ref), k
        else:
            assert relerr(st.w, ref) <= 1e-10, (k, relerr(st.w, ref))
    assert st.n == m["n"] and st.t == m["t"]
    assert abs(st.inner_iterations - m["inner"]) <= max(1, 0.05 * m["inner"])
    # the solver's operator is the reference's A = I - (dt^2/2) L_h
    x = ARR[f"{key}__v0"]
    np.testing.assert_allclose(solver.apply(x), x - 0.5 * corr.dt**2 * op.apply_values(x), rtol=0, atol=1e-14)
