"""Small runs of every kernel family in one process (explicit wavefront / two-step / one-step / general kernels, slabs with
two-step passes, batched frequencies, GMRES vectors, implicit CG + multigrid
+ tridiagonal).  Exits 0 and prints one line per case.  (compute-sanitizer
is not available on the GPU pool; out-of-bounds safety rests on the parity
tests against the CPU reference at ragged sizes.)"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2504_03074_b200 as wh  # noqa: E402
from paper_2504_03074_b200 import _native  # noqa: E402
from paper_2504_03074_b200.slab import DeviceShard, LocalHalo, exchange_forcing, run_local_solve, slab_ranges  # noqa: E402


def explicit(dim, cells, bcs="dirichlet", order=2, omega=9.0):
    g = wh.build_grid(dim, [(0.0, 1.0)] * dim, cells, bcs)
    f = wh.multi_gaussian_source(g, omega, 2, seed=1)
    prob = wh.HelmholtzProblem(g, order, 1.0, omega, f)
    cfg = wh.FilterConfig(omega=omega, mode="explicit")
    v, run = wh.fpi_solve(prob, cfg, tol=-1.0, maxit=2)
    x, krun = wh.krylov_solve(prob, cfg, tol=1e-6, restart=4, maxit=8)
    print("explicit", dim, cells, bcs, order, float(np.abs(v.values).max()), krun.iterations, flush=True)


def slabs(cells, nslabs, omega=7.0):
    d = len(cells)
    g = wh.build_grid(d, [(0.0, 1.0)] * d, cells, "dirichlet")
    f = np.asarray(wh.multi_gaussian_source(g, omega, 2, seed=2).values)
    corr = wh.correct_explicit(omega, g, 2, 1.0)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    sched = wh.time_schedule(corr, cfg)
    rng = slab_ranges(g.shape[0], nslabs)
    shards = [DeviceShard(g, r) for r in rng]
    for sh, (p0, p1) in zip(shards, rng):
        sh.set_schedule(sched)
        sh.upload(_native.F, np.ascontiguousarray(f[p0:p1]))
        sh.zero(_native.V)
    halo = LocalHalo(shards)
    exchange_forcing(shards, halo)
    s = [sum(run_local_solve(shards, halo)) for _ in range(2)]
    print("slabs", cells, nslabs, s[-1], flush=True)
    for sh in shards:
        sh.ctx.close()


def batched():
    from paper_2504_03074_b200.batch import fpi_solve_batched

    g = wh.build_grid(2, [(0.0, 1.0)] * 2, (40, 36), "dirichlet")
    f = wh.multi_gaussian_source(g, 10.0, 2, seed=3)
    out = fpi_solve_batched(g, f, [5.0, 9.0, 13.0], tol=-1.0, maxit=2)
    print("batched", len(out), flush=True)


def implicit(dim, cells, bcs="dirichlet", order=2, omega=8.0, n_t=8):
    g = wh.build_grid(dim, [(0.0, 1.0)] * dim, cells, bcs)
    f = wh.multi_gaussian_source(g, omega, 2, seed=4)
    prob = wh.HelmholtzProblem(g, order, 1.0, omega, f)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=n_t, mode="implicit")
    v, run = wh.fpi_solve(prob, cfg, tol=-1.0, maxit=2)
    x, krun = wh.krylov_solve(prob, cfg, tol=1e-6, restart=4, maxit=6)
    print("implicit", dim, cells, bcs, order, run.inner_iterations, krun.iterations, flush=True)


if __name__ == "__main__":
    explicit(2, (64, 48))
    explicit(3, (24, 20, 28))
    explicit(1, (50,))
    explicit(2, (30, 26), "periodic", 4)
    slabs((40, 30), 3)
    slabs((20, 18, 22), 3)
    batched()
    implicit(2, (64, 64))
    implicit(2, (128, 64), order=4)
    implicit(1, (64,))
    implicit(1, (48,), order=4)
    implicit(3, (10, 12, 8))
    implicit(2, (24, 20), "periodic")
    print("all paths done")
