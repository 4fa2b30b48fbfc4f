"""Golden fixtures for the implicit (trapezoidal) path, produced by the REAL
reference package (this container only):

    python tests/golden/make_golden_implicit.py        # ~1 min

Each case stores its inputs (forcing f, start field v0) and the reference's
outputs: W(v0, f) from ``wave_solve_filtered`` in implicit mode with the
reference's own ``make_implicit_solver`` (timestep.py:183-247: tridiagonal /
multigrid-preconditioned CG / plain CG), the inner iteration count, and for
some cases 3 fixed-point iterates (the ``_iterate`` body, driver.py:215-230)
or a GMRES solve (``krylov_solve``, driver.py:273-300).  Written to
tests/golden/implicit.npz + implicit.json.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import reference_harness as RH  # noqa: E402

# name: (dim, cells, bcs, order, omega, n_t, extra)
CASES = {
    "mg2d_64": (2, (64, 64), "dirichlet", 2, 11.0, 10, {"fpi": 3}),
    "mg2d_32x40": (2, (32, 40), "dirichlet", 2, 9.0, 8, {}),
    "cg2d_30": (2, (30, 30), "dirichlet", 2, 7.0, 10, {}),          # 30 -> 15: no hierarchy, plain CG
    "mg2d_p4": (2, (32, 32), "dirichlet", 4, 8.0, 10, {}),         # order 4, V-cycle of the p=2 operator
    "mg2d_8": (2, (8, 8), "dirichlet", 2, 5.5, 6, {}),             # single-level hierarchy
    "tri1d_p2": (1, (64,), "dirichlet", 2, 6.0, 10, {"fpi": 3}),  # direct tridiagonal solve
    "tri1d_p4": (1, (48,), "dirichlet", 4, 6.0, 7, {}),           # tridiagonal-preconditioned CG
    "cg3d": (3, (10, 12, 8), "dirichlet", 2, 5.0, 6, {}),         # plain CG (3D)
    "cg2d_per": (2, (24, 20), "periodic", 2, 6.5, 9, {}),         # periodic: plain CG
    "mg2d_expl_first": (2, (32, 32), "dirichlet", 2, 10.0, 5, {"implicit_first_step": False}),
    "gmres2d": (2, (32, 32), "dirichlet", 2, 5.5, 10, {"gmres": True}),
}


def main():
    wh = RH.import_reference()
    arrays, meta = {}, {}
    for name, (dim, cells, bcs, order, omega, n_t, extra) in CASES.items():
        g = RH.grid(dim, [(0.0, 1.0)] * dim, cells, bcs)
        rng = np.random.default_rng(sum(name.encode()))
        f = RH.multi_gaussian(g, omega, 3, seed=len(name)).values
        v0 = wh.grid.GridField.from_values(g, rng.standard_normal(g.shape) * 1e-2).values
        corr = wh.timestep.correct_implicit(omega, n_t)
        cfg = wh.filters.FilterConfig(omega=omega, periods=1, steps_per_period=n_t, mode="implicit")
        op = wh.grid.DiscreteOperator(g, order, 1.0)
        solver = wh.timestep.make_implicit_solver(op, corr.dt)
        fld = wh.grid.GridField.from_values
        first = extra.get("implicit_first_step", True)
        out = wh.timestep.wave_solve_filtered(fld(g, v0), fld(g, f), cfg, corr, op, linear_solver=solver,
                                              implicit_first_step=first).values
        arrays[f"{name}/f"] = f
        arrays[f"{name}/v0"] = v0
        arrays[f"{name}/out"] = out
        m = {"dim": dim, "cells": list(cells), "bcs": bcs, "order": order, "omega": omega, "n_t": n_t,
             "implicit_first_step": first, "inner": solver.inner,
             "precond": ("tri" if solver._tri is not None else ("mg" if solver._mg is not None else None))}
        if extra.get("fpi"):
            solver = wh.timestep.make_implicit_solver(op, corr.dt)
            v = wh.grid.GridField.zeros(g, ghost=max(2, op.ghost_width))
            res = []
            for k in range(extra["fpi"]):
                v_new = wh.timestep.wave_solve_filtered(v, fld(g, f), cfg, corr, op, linear_solver=solver)
                res.append(float(np.linalg.norm(v_new.values - v.values) / math.sqrt(g.size)))
                v = v_new
                arrays[f"{name}/fpi{k + 1}"] = np.array(v.values)
            m["fpi_residuals"] = res
        if extra.get("gmres"):
            prob = wh.driver.HelmholtzProblem(g, order, 1.0, omega, fld(g, f))
            x, run = wh.driver.krylov_solve(prob, cfg, tol=1e-9, restart=10)
            arrays[f"{name}/gmres_x"] = np.array(x.values)
            m["gmres"] = {"iterations": run.iterations, "residuals": run.residuals, "tol": 1e-9, "restart": 10}
        meta[name] = m
        print(name, m["precond"], m["inner"], flush=True)
    np.savez_compressed(os.path.join(HERE, "implicit.npz"), **arrays)
    with open(os.path.join(HERE, "implicit.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
