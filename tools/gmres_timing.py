"""GMRES (krylov_solve) cost split on one GPU: total time vs the mat-vecs alone.

    python tools/gmres_timing.py --cells 2048 --omega 100.5 --restart 20 --maxit 20
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=2048)
    ap.add_argument("--omega", type=float, default=100.5)
    ap.add_argument("--restart", type=int, default=20)
    ap.add_argument("--maxit", type=int, default=20)
    a = ap.parse_args()
    import paper_2504_03074_b200 as wh
    from paper_2504_03074_b200 import _native
    from paper_2504_03074_b200 import timestep as ts
    from paper_2504_03074_b200.device import device_problem

    ts._COURANT[2] = 0.9
    g = wh.build_grid(2, [(0.0, 1.0)] * 2, [a.cells] * 2, "dirichlet")
    f = wh.multi_gaussian_source(g, a.omega, 8, seed=0)
    prob = wh.HelmholtzProblem(g, 2, 1.0, a.omega, f)
    cfg = wh.FilterConfig(omega=a.omega, mode="explicit")
    wh.krylov_solve(prob, cfg, tol=0.0, restart=a.restart, maxit=2)
    dp = device_problem(g)
    dp.ctx.synchronize()
    t0 = time.perf_counter()
    x, run = wh.krylov_solve(prob, cfg, tol=0.0, restart=a.restart, maxit=a.maxit)
    dp.ctx.synchronize()
    tot = time.perf_counter() - t0
    ids = dp.ctx.vec_reserve(2)
    dp.ctx.vec_upload(ids[0], f.values)
    dp.ctx.matvec(ids[0], ids[1])
    dp.ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.maxit):
        dp.ctx.matvec(ids[0], ids[1])
    dp.ctx.synchronize()
    mv = time.perf_counter() - t0
    print(json.dumps({"grid": list(g.shape), "restart": a.restart, "iterations": run.iterations,
                      "total_ms": tot * 1e3, "matvecs_ms": mv * 1e3, "vector_work_share": 1 - mv / tot}))


if __name__ == "__main__":
    main()
