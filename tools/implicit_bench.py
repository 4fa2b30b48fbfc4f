"""Implicit-mode timing on one GPU: implicit WaveHoltz iterations (CG + multigrid
V-cycle per trapezoidal step) and the V-cycle alone.

    python tools/implicit_bench.py --cells 1024 --nt 20 --iters 3
"""

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=1024)
    ap.add_argument("--omega", type=float, default=50.5)
    ap.add_argument("--nt", type=int, default=20)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--vcycles", type=int, default=50)
    a = ap.parse_args()

    import torch

    import paper_2504_03074_b200 as wh
    from paper_2504_03074_b200.device import device_problem
    from paper_2504_03074_b200.implicit import implicit_solver_for

    g = wh.build_grid(2, [(0.0, 1.0)] * 2, [a.cells] * 2, "dirichlet")
    f = wh.multi_gaussian_source(g, a.omega, 4, seed=0)
    prob = wh.HelmholtzProblem(g, 2, 1.0, a.omega, f)
    cfg = wh.FilterConfig(omega=a.omega, periods=1, steps_per_period=a.nt, mode="implicit")
    corr = wh.correct_implicit(a.omega, a.nt)
    dp = device_problem(g)
    s = implicit_solver_for(dp, g, 2, 1.0, corr.dt)
    ctx = dp.ctx
    out = {"grid": list(g.shape), "omega": a.omega, "N_t": a.nt, "precond": s.precond}

    # V-cycle alone (graph replay)
    r, z = s.r, s.z
    ctx.vec_upload(r, np.random.default_rng(0).standard_normal(g.shape))
    for _ in range(3):
        ctx.mg_vcycle(r, z)
    ctx.synchronize()
    l0 = ctx.launch_count()
    t0 = time.perf_counter()
    for _ in range(a.vcycles):
        ctx.mg_vcycle(r, z)
    ctx.synchronize()
    dt = (time.perf_counter() - t0) / a.vcycles
    out["vcycle_us"] = dt * 1e6
    out["vcycle_launches"] = (ctx.launch_count() - l0) / a.vcycles

    # implicit FPI iterations (warm-up 1)
    wh.fpi_solve(prob, cfg, tol=-1.0, maxit=1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v, run = wh.fpi_solve(prob, cfg, tol=-1.0, maxit=a.iters)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out["iter_ms"] = dt * 1e3 / a.iters
    out["gpts"] = g.size * a.nt * a.iters / dt / 1e9
    out["cg_iters_per_step"] = run.inner_iterations / (a.iters * a.nt)
    out["residuals"] = run.residuals
    print(json.dumps(out))


if __name__ == "__main__":
    main()
