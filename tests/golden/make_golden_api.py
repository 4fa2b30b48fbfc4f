"""Golden outputs of the reference's host-callable API that sits beside the hot path:
``linalg.gmres_solve`` (linalg.py:102-183) on seeded operators, ``timestep.step_implicit`` with
``make_implicit_solver`` (timestep.py:148-247).  Run where /root/reference exists:

    python tests/golden/make_golden_api.py        # writes tests/golden/api.{json,npz}
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import reference_harness as RH  # noqa: E402


def main():
    wh = RH.import_reference()
    import waveholtz.linalg as L
    import waveholtz.timestep as T

    rng = np.random.default_rng(77)
    meta, arr = {}, {}
    n = 120
    A = np.eye(n) * 4.0 + rng.standard_normal((n, n)) * (0.6 / np.sqrt(n))
    b = rng.standard_normal(n)
    x0 = rng.standard_normal(n) * 0.1
    arr["A"], arr["b"], arr["x0"] = A, b, x0
    for key, kw in (("dense", {}), ("dense_x0", {"x0": x0}), ("dense_atol", {"atol": 1e-6, "tol": 0.0})):
        x, rep = L.gmres_solve(A, b, restart=12, maxit=200, **{"tol": 1e-10, **kw})
        arr[f"{key}__x"] = x
        meta[key] = {"iterations": rep.iterations, "converged": bool(rep.converged),
                     "relative_residual": rep.relative_residual, "work_units": rep.work_units,
                     "history": [float(h) for h in rep.residual_history]}
    # callable on a 2D array
    shp = (20, 30)
    D = 3.0 + rng.random(shp)
    B = rng.standard_normal(shp)

    def op(v):
        out = D * v
        out[1:, :] += 0.3 * v[:-1, :]
        out[:, :-1] -= 0.2 * v[:, 1:]
        return out

    arr["D"], arr["B"] = D, B
    x, rep = L.gmres_solve(op, B, tol=1e-11, restart=25, maxit=300)
    arr["callable__x"] = x
    meta["callable"] = {"iterations": rep.iterations, "converged": bool(rep.converged),
                        "history": [float(h) for h in rep.residual_history]}
    # step_implicit / make_implicit_solver: 1D p = 2 (tridiagonal) and 2D (MG-PCG), 5 steps
    for key, dim, cells, order in (("imp1d", 1, [64], 2), ("imp2d", 2, [32, 32], 2), ("imp1d_p4", 1, [48], 4)):
        g = RH.grid(dim, [(0.0, 1.0)] * dim, cells)
        op_ = wh.grid.DiscreteOperator(g, order, 1.0)
        corr = T.correct_implicit(9.5, 12)
        f = RH.multi_gaussian(g, 9.5, 2, seed=5).values
        v0 = rng.standard_normal(g.shape) * 1e-2
        v0 = wh.grid.GridField.from_values(g, v0).values
        solver = T.make_implicit_solver(op_, corr.dt, tol=1e-12)
        st = T.WaveState.start(np.array(v0))
        outs = []
        for _ in range(5):
            st = T.step_implicit(st, op_, np.array(f), corr, solver)
            outs.append(np.array(st.w))
        arr[f"{key}__f"], arr[f"{key}__v0"] = np.array(f), np.array(v0)
        arr[f"{key}__w"] = np.stack(outs)
        meta[key] = {"dim": dim, "cells": cells, "order": order, "omega": 9.5, "n_t": 12,
                     "inner": int(st.inner_iterations), "t": st.t, "n": st.n}
    json.dump(meta, open(os.path.join(HERE, "api.json"), "w"), indent=1)
    np.savez_compressed(os.path.join(HERE, "api.npz"), **arr)
    print("wrote api")


if __name__ == "__main__":
    main()
