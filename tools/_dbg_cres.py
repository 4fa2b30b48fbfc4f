"""Debug: cluster-resident kernel vs the C oracle on small grids; prints where results differ."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2504_03074_b200 as wh
from paper_2504_03074_b200 import timestep as ts
from oracle import native as ON, waveholtz_oracle as O
ts._COURANT[2] = 0.9
for cells, omega, nit in [((128, 128), 20.3, 1), ((128, 128), 20.3, 2), ((256, 256), 40.0, 1), ((32, 32), 7.0, 1),
                          ((32, 32), 7.3, 1), ((16, 16), 5.0, 1)]:
    g = wh.build_grid(2, [(0.0, 1.0)] * 2, list(cells), "dirichlet")
    f = wh.multi_gaussian_source(g, omega, 4, seed=1)
    corr = wh.correct_explicit(omega, g, 2, 1.0)
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    v0 = np.random.default_rng(11).standard_normal(g.shape) * 1e-3
    v = wh.GridField.from_values(g, v0)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    if nit == 1:
        got = wh.wave_solve_filtered(v, f, cfg, corr, wh.DiscreteOperator(g, 2, 1.0)).values
        ref = ON.wave_solve(np.array(v.values), np.array(f.values), g.spacing, sc)
    else:
        prob = wh.HelmholtzProblem(g, 2, 1.0, omega, f)
        got = wh.fpi_solve(prob, cfg, tol=-1.0, maxit=nit)[0].values
        ref, _ = ON.fpi(np.array(f.values), g.spacing, sc, nit)
    dp = wh.device.device_problem(g)
    bad = got != ref
    rows = np.where(bad.any(axis=1))[0]
    err = np.max(np.abs(got - ref)) / max(1e-300, np.max(np.abs(ref)))
    print(cells, "N_t", corr.steps_per_period, "iters", nit, "plan", dp.ctx.plan(), "bad", int(bad.sum()),
          "relerr %.3e" % err, "bad rows", rows[:20].tolist(), "...", rows[-5:].tolist())
    wh.release_device_cache()
