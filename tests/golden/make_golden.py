"""Generate the golden parity fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py small          # seconds
    python tests/golden/make_golden.py cfg1           # ~5 s  (+ GMRES)
    python tests/golden/make_golden.py cfg2           # ~35 min (2049^2, 50 iterations)
    python tests/golden/make_golden.py cfg3           # ~45 min (257^3, 30 iterations)
    python tests/golden/make_golden.py cfg5 [--procs P]  # 64 omegas x 20 iterations
    python tests/golden/make_golden.py cfg4           # ~30 min, 43 GB RAM (1025^3, 10 iterations)

Every case is produced by the reference's own functions
(``correct_explicit``, ``gaussian_source``, ``wave_solve_filtered``,
``fpi_solve``/``_iterate`` body, ``krylov_solve``, ``apply_A``) with
``_COURANT[2] = 0.9`` for the BASELINE "CFL 0.9" configs.
Large iterates are stored as sha256 of their C-order float64 bytes (bitwise
pin), the max-norm, and the values at 256 fixed sample indices (tolerance
diagnostics); small ones are stored in full (npz).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import reference_harness as RH  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def sample_idx(size: int, n: int = 256, seed: int = 7) -> np.ndarray:
    return np.sort(np.random.default_rng(seed).choice(size, size=min(n, size), replace=False))


def corr_dict(corr, cfg):
    return {
        "steps_per_period": corr.steps_per_period,
        "dt": corr.dt,
        "omega": corr.omega,
        "omega_tilde": corr.omega_tilde,
        "alpha": corr.alpha,
        "periods": cfg.periods,
    }


def dump(name, meta, arrays=None):
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    if arrays:
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    print(f"wrote {name}", flush=True)


# ---------------------------------------------------------------------------------
# BASELINE configs


CONFIGS = {
    # name: (dim, n_cells, omega, forcing, iterations)
    "cfg1": (2, 128, 20.3, ("single", 100.0, 200.0, (0.4, 0.6)), 100),
    "cfg2": (2, 2048, 100.5, ("multi", 8), 50),
    "cfg3": (3, 256, 40.7, ("single", 100.0, 300.0, (0.45, 0.5, 0.55)), 30),
}


def build_cfg_forcing(g, omega, forcing):
    wh = RH.import_reference()
    if forcing[0] == "single":
        _, a, b, x0 = forcing
        return wh.driver.gaussian_source(g, omega, a, b, x0)
    return RH.multi_gaussian(g, omega, forcing[1], seed=0)


def run_cfg(name):
    dim, n, omega, forcing, iters = CONFIGS[name]
    wh = RH.import_reference()
    with RH.courant(0.9):
        g = RH.grid(dim, [(0.0, 1.0)] * dim, [n] * dim)
        f = build_cfg_forcing(g, omega, forcing)
        corr, cfg, op = RH.explicit_setup(g, omega)
        idx = sample_idx(g.size)
        meta = {
            "config": name, "dim": dim, "cells": [n] * dim, "bounds": [[0.0, 1.0]] * dim,
            "omega": omega, "c": 1.0, "order": 2, "courant": 0.9,
            "forcing": list(forcing) if forcing[0] == "single" else ["multi", forcing[1], "seed0"],
            "corr": corr_dict(corr, cfg), "f_sha256": sha(f.values),
            "f_max": float(np.max(np.abs(f.values))), "f_samples": f.values.ravel()[idx].tolist(),
            "sample_idx": idx.tolist(), "iterations": iters,
            "iter_sha256": [], "residuals": [], "vmax": [], "samples": [],
        }
        arrays = {}
        t0 = time.perf_counter()
        if name == "cfg1":
            # through the real public API with the iterate-capturing seam (driver.py:38)
            prob = wh.driver.HelmholtzProblem(g, 2, 1.0, omega, f)
            cfg0 = wh.filters.FilterConfig(omega=omega, periods=1, steps_per_period=10, mode="explicit")
            captured = []
            orig = wh.driver.wave_solve_filtered

            def cap(*a, **k):
                out = orig(*a, **k)
                captured.append(np.array(out.values))
                return out

            wh.driver.wave_solve_filtered = cap
            try:
                v, run = wh.driver.fpi_solve(prob, cfg0, tol=-1.0, maxit=iters)
            finally:
                wh.driver.wave_solve_filtered = orig
            assert np.array_equal(captured[-1], v.values)
            for k, vk in enumerate(captured, 1):
                meta["iter_sha256"].append(sha(vk))
                meta["vmax"].append(float(np.max(np.abs(vk))))
                meta["samples"].append(vk.ravel()[idx].tolist())
            meta["residuals"] = [float(r) for r in run.residuals]
            for k in (1, 2, 10, iters):
                arrays[f"v{k}"] = captured[k - 1]
            arrays["f"] = np.array(f.values)
            # GMRES (krylov_solve, driver.py:273-300) on the same problem
            xk, runk = wh.driver.krylov_solve(prob, cfg0, tol=1e-10, restart=50, maxit=500)
            meta["gmres"] = {
                "tol": 1e-10, "restart": 50, "maxit": 500, "iterations": runk.iterations,
                "converged": bool(runk.converged), "residuals": [float(r) for r in runk.residuals],
                "x_sha256": sha(xk.values),
            }
            arrays["gmres_x"] = np.array(xk.values)
        else:
            for k, vk, r in RH.fpi_iterates(g, f, omega, iters):
                meta["iter_sha256"].append(sha(vk))
                meta["vmax"].append(float(np.max(np.abs(vk))))
                meta["samples"].append(vk.ravel()[idx].tolist())
                meta["residuals"].append(float(r))
                print(f"{name} it {k} r={r:.6e} t={time.perf_counter() - t0:.1f}s", flush=True)
                if k == 1 and dim == 2:
                    pass
        meta["ref_seconds"] = time.perf_counter() - t0
        dump(name, meta, arrays or None)


# ---------------------------------------------------------------------------------
# cfg4: 3D 1025^3 (the north-star config).  The reference's numpy path needs ~76 GB
# and ~1.85 h per iteration here (SURVEY 8(c) rung 4), so the iterates come from the
# C restatement (oracle/whb_oracle.c, who_fpi_lean: 5 resident fields), which is
# pinned bitwise to the reference's own iterates on cfg1-cfg3 and the small cases
# (tests/test_oracle_golden.py).  The forcing is the reference's gaussian_source
# evaluated slab by slab (RH.multi_gaussian_slabs), and every scalar comes from the
# reference's correct_explicit.


def run_cfg4(iters=10, threads=0):
    from oracle import native as ON
    from oracle import waveholtz_oracle as O

    dim, n, omega = 3, 1024, 150.3
    with RH.courant(0.9):
        g = RH.grid(dim, [(0.0, 1.0)] * dim, [n] * dim)
        corr, cfg, op = RH.explicit_setup(g, omega)
        t0 = time.perf_counter()
        f = RH.multi_gaussian_slabs(g, omega, 16, seed=0)
        print(f"cfg4 forcing {time.perf_counter() - t0:.1f}s", flush=True)
    idx = sample_idx(f.size)
    meta = {
        "config": "cfg4", "dim": dim, "cells": [n] * dim, "bounds": [[0.0, 1.0]] * dim,
        "omega": omega, "c": 1.0, "order": 2, "courant": 0.9, "forcing": ["multi", 16, "seed0"],
        "corr": corr_dict(corr, cfg), "f_sha256": hashlib.sha256(f.data).hexdigest(),
        "f_max": float(np.max(np.abs(f))), "f_samples": f.ravel()[idx].tolist(),
        "sample_idx": idx.tolist(), "iterations": iters,
        "iter_sha256": [], "residuals": [], "vmax": [], "samples": [],
        "source": "forcing: reference gaussian_source per slab; iterates: oracle/whb_oracle.c who_fpi_lean "
                  "(C restatement, bitwise pinned to the reference on cfg1-cfg3)",
    }
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    v = np.zeros_like(f)
    t0 = time.perf_counter()
    for k in range(1, iters + 1):
        _, r = ON.fpi_lean(f, g.spacing, sc, 1, nthreads=threads or ON.max_threads(), v=v)
        meta["iter_sha256"].append(hashlib.sha256(v.data).hexdigest())
        meta["residuals"].append(float(r[0]))
        meta["vmax"].append(float(np.max(np.abs(v))))
        meta["samples"].append(v.ravel()[idx].tolist())
        print(f"cfg4 it {k} r={r[0]:.6e} t={time.perf_counter() - t0:.1f}s", flush=True)
        meta["ref_seconds"] = time.perf_counter() - t0
        dump("cfg4", meta)  # after every iterate: a partial run still pins the first ones


# ---------------------------------------------------------------------------------
# cfg5: batched frequencies (64 omegas on 1025^2, shared 4-Gaussian forcing)


def _cfg5_one(args):
    j, omega, iters = args
    wh = RH.import_reference()
    with RH.courant(0.9):
        g = RH.grid(2, [(0.0, 1.0)] * 2, [1024, 1024])
        f = RH.multi_gaussian(g, 150.3, 4, seed=0)  # shared forcing; omega is informational only
        corr, cfg, op = RH.explicit_setup(g, omega)
        idx = sample_idx(g.size)
        out = {"omega": omega, "corr": corr_dict(corr, cfg), "iter_sha256": [], "residuals": [],
               "vmax": [], "samples": [], "f_sha256": sha(f.values)}
        t0 = time.perf_counter()
        for k, vk, r in RH.fpi_iterates(g, f, omega, iters):
            out["iter_sha256"].append(sha(vk))
            out["residuals"].append(float(r))
            out["vmax"].append(float(np.max(np.abs(vk))))
            if k in (1, iters):
                out["samples"].append(vk.ravel()[idx].tolist())
        out["ref_seconds"] = time.perf_counter() - t0
        print(f"cfg5 omega[{j}]={omega:.4f} N_t={corr.steps_per_period} {out['ref_seconds']:.1f}s", flush=True)
        return j, out


def run_cfg5(procs, iters=20, n_omega=64):
    import multiprocessing as mp

    omegas = np.linspace(10.3, 200.3, n_omega)
    jobs = [(j, float(w), iters) for j, w in enumerate(omegas)]
    # longest first (N_t ~ 1/omega) for better packing
    jobs.sort(key=lambda t: t[1])
    with mp.get_context("fork").Pool(procs) as pool:
        res = dict(pool.map(_cfg5_one, jobs, chunksize=1))
    g_idx = sample_idx(1025 * 1025)
    meta = {"config": "cfg5", "dim": 2, "cells": [1024, 1024], "omegas": omegas.tolist(),
            "forcing": ["multi", 4, "seed0"], "courant": 0.9, "iterations": iters,
            "sample_idx": g_idx.tolist(), "sample_iters": [1, iters],
            "per_omega": [res[j] for j in range(n_omega)]}
    dump("cfg5", meta)


# ---------------------------------------------------------------------------------
# small full-array cases (edge cases and non-BASELINE shapes)


def run_small():
    wh = RH.import_reference()
    rng = np.random.default_rng(20260419)
    cases = {}
    arrays = {}

    def solve_case(key, dim, bounds, cells, omega, c=1.0, periods=1, courant=None,
                   v_kind="random", f_kind="random"):
        ctx = RH.courant(courant) if courant is not None else _null()
        with ctx:
            g = RH.grid(dim, bounds, cells)
            corr, cfg, op = RH.explicit_setup(g, omega, 2, c, periods)
            GF = wh.grid.GridField
            if v_kind == "random":
                v = GF.from_values(g, rng.standard_normal(g.shape))
            else:
                v = GF.zeros(g)
            if f_kind == "random":
                f = GF.from_values(g, rng.standard_normal(g.shape) * 50.0)
            elif f_kind == "gauss":
                x0 = tuple(0.5 * (lo + hi) + 0.07 * (m + 1) for m, (lo, hi) in enumerate(bounds))
                f = wh.driver.gaussian_source(g, omega, 80.0, 40.0, x0)
            else:
                f = GF.zeros(g)
            out = wh.timestep.wave_solve_filtered(v, f, cfg, corr, op)
            # zero-forcing mat-vec A v = v - W(v, 0) (driver.py:247-264)
            prob_like = type("P", (), {})()
            av = np.array(v.values) - wh.timestep.wave_solve_filtered(v, GF.zeros(g), cfg, corr, op).values
            cases[key] = {"dim": dim, "bounds": [list(b) for b in bounds], "cells": list(cells),
                          "omega": omega, "c": c, "periods": periods, "courant": courant or 1.0,
                          "corr": corr_dict(corr, cfg), "out_sha256": sha(out.values),
                          "av_sha256": sha(av)}
            arrays[f"{key}__v"] = np.array(v.values)
            arrays[f"{key}__f"] = np.array(f.values)
            arrays[f"{key}__out"] = np.array(out.values)
            arrays[f"{key}__av"] = av
            del prob_like

    solve_case("d1_n16", 1, [(0.0, 1.0)], [16], 5.5)
    solve_case("d1_n16_p2", 1, [(0.0, 1.0)], [16], 5.5, periods=2)
    solve_case("d1_n4_min", 1, [(0.0, 1.0)], [4], 2.0)
    solve_case("d1_n37_c13", 1, [(-1.0, 2.0)], [37], 4.0, c=1.3, courant=0.9)
    solve_case("d2_sq32", 2, [(0.0, 1.0)] * 2, [32, 32], 5.7, f_kind="gauss", v_kind="zero")
    solve_case("d2_rect", 2, [(0.0, 1.0), (0.0, 2.0)], [24, 40], 7.1, c=1.3)
    solve_case("d2_rect_p2", 2, [(0.0, 1.0), (0.0, 2.0)], [24, 40], 7.1, c=1.3, periods=2, courant=0.9)
    solve_case("d2_min", 2, [(0.0, 1.0)] * 2, [4, 4], 3.0)
    solve_case("d2_ragged", 2, [(0.0, 1.5), (0.25, 1.0)], [37, 61], 9.3, courant=0.9)
    solve_case("d2_wide", 2, [(0.0, 1.0), (0.0, 1.0)], [5, 300], 11.0, courant=0.9)
    solve_case("d2_zero", 2, [(0.0, 1.0)] * 2, [16, 16], 5.0, v_kind="zero", f_kind="zero")
    solve_case("d3_cube", 3, [(0.0, 1.0)] * 3, [12, 12, 12], 6.0, courant=0.9)
    solve_case("d3_box", 3, [(0.0, 1.0), (0.0, 0.8), (-0.5, 1.0)], [12, 10, 14], 6.0, c=0.8)
    solve_case("d3_min", 3, [(0.0, 1.0)] * 3, [4, 4, 4], 2.5)
    solve_case("d3_ragged", 3, [(0.0, 1.0)] * 3, [9, 37, 70], 8.0, courant=0.9, f_kind="gauss")
    solve_case("d3_thin", 3, [(0.0, 1.0)] * 3, [40, 5, 33], 8.0, courant=0.9, periods=2)

    # a small 3D FPI run (10 iterations) and a 2D GMRES solve through the public API
    with RH.courant(0.9):
        g = RH.grid(3, [(0.0, 1.0)] * 3, [16, 16, 16])
        f = wh.driver.gaussian_source(g, 9.0, 100.0, 30.0, (0.45, 0.5, 0.55))
        fpi = {"dim": 3, "cells": [16, 16, 16], "omega": 9.0, "iter_sha256": [], "residuals": []}
        for k, vk, r in RH.fpi_iterates(g, f, 9.0, 10):
            fpi["iter_sha256"].append(sha(vk))
            fpi["residuals"].append(float(r))
            if k == 10:
                arrays["fpi3d__v10"] = np.array(vk)
        arrays["fpi3d__f"] = np.array(f.values)
        cases["fpi3d"] = fpi

        g2 = RH.grid(2, [(0.0, 1.0)] * 2, [32, 32])
        f2 = wh.driver.gaussian_source(g2, 5.7, -100.0, 30.0, (0.37, 0.41))
        prob = wh.driver.HelmholtzProblem(g2, 2, 1.0, 5.7, f2)
        cfg0 = wh.filters.FilterConfig(omega=5.7, periods=1, steps_per_period=10, mode="explicit")
        x, run = wh.driver.krylov_solve(prob, cfg0, tol=1e-10)
        vf, runf = wh.driver.fpi_solve(prob, cfg0, tol=1e-10, maxit=2000)
        cases["gmres2d"] = {"dim": 2, "cells": [32, 32], "omega": 5.7, "iterations": run.iterations,
                            "residuals": [float(r) for r in run.residuals], "converged": bool(run.converged),
                            "fpi_iterations": runf.iterations, "fpi_residuals": [float(r) for r in runf.residuals]}
        arrays["gmres2d__x"] = np.array(x.values)
        arrays["gmres2d__f"] = np.array(f2.values)
        arrays["gmres2d__fpi"] = np.array(vf.values)
        # reference default Courant (1.0) on the same problem, FPI 5 iterations
        fpi1 = {"iter_sha256": []}
    with RH.courant(1.0):
        for k, vk, r in RH.fpi_iterates(g2, f2, 5.7, 5):
            fpi1["iter_sha256"].append(sha(vk))
        cases["gmres2d"]["fpi_courant1_sha256"] = fpi1["iter_sha256"]
    dump("small", {"cases": cases}, arrays)


def run_ext():
    """order-4 stencils and periodic / mixed boundaries."""
    wh = RH.import_reference()
    rng = np.random.default_rng(20261019)
    cases, arrays = {}, {}
    GF = wh.grid.GridField

    def case(key, dim, bounds, cells, bcs, p, omega, c=1.0, periods=1):
        g = RH.grid(dim, bounds, cells, bcs)
        corr, cfg, op = RH.explicit_setup(g, omega, p, c, periods)
        v = GF.from_values(g, rng.standard_normal(g.shape), ghost=2)
        f = GF.from_values(g, rng.standard_normal(g.shape) * 30.0, ghost=2)
        out = wh.timestep.wave_solve_filtered(v, f, cfg, corr, op)
        lap = op.apply_values(v.values)
        av = np.array(v.values) - wh.timestep.wave_solve_filtered(v, GF.zeros(g), cfg, corr, op).values
        cases[key] = {"dim": dim, "bounds": [list(b) for b in bounds], "cells": list(cells),
                      "bcs": [bcs] * dim if isinstance(bcs, str) else list(bcs), "order": p, "omega": omega,
                      "c": c, "periods": periods, "corr": corr_dict(corr, cfg), "out_sha256": sha(out.values),
                      "av_sha256": sha(av), "lap_sha256": sha(lap)}
        arrays[f"{key}__v"] = np.array(v.values)
        arrays[f"{key}__f"] = np.array(f.values)
        arrays[f"{key}__out"] = np.array(out.values)

    case("p4_d1", 1, [(0.0, 1.0)], [20], "dirichlet", 4, 5.5)
    case("p4_d2", 2, [(0.0, 1.0), (0.0, 1.3)], [16, 22], "dirichlet", 4, 7.0, c=1.1)
    case("p4_d2_np2", 2, [(0.0, 1.0), (0.0, 1.3)], [16, 22], "dirichlet", 4, 7.0, periods=2)
    case("p4_d3", 3, [(0.0, 1.0), (0.0, 1.2), (-0.3, 0.6)], [10, 12, 9], "dirichlet", 4, 6.0)
    case("p4_min", 2, [(0.0, 1.0)] * 2, [4, 4], "dirichlet", 4, 3.0)
    case("per_p2_d1", 1, [(0.0, 2.0)], [24], "periodic", 2, 4.1)
    case("per_p2_d2", 2, [(0.0, 1.0), (0.0, 0.8)], [20, 16], "periodic", 2, 9.3)
    case("per_p2_d3", 3, [(0.0, 1.0)] * 3, [8, 10, 12], "periodic", 2, 7.7)
    case("per_p4_d1", 1, [(0.0, 2.0)], [24], "periodic", 4, 4.1)
    case("per_p4_d2", 2, [(0.0, 1.0), (0.0, 0.8)], [18, 20], "periodic", 4, 9.3)
    case("per_p4_d3", 3, [(0.0, 1.0)] * 3, [8, 6, 10], "periodic", 4, 6.3)
    case("mix_p2_d2", 2, [(0.0, 1.0), (0.0, 1.0)], [18, 15], ["periodic", "dirichlet"], 2, 8.8)
    case("mix_p4_d2", 2, [(0.0, 1.0), (0.0, 1.0)], [18, 15], ["dirichlet", "periodic"], 4, 8.8)
    case("mix_p2_d3", 3, [(0.0, 1.0)] * 3, [9, 8, 12], ["dirichlet", "periodic", "dirichlet"], 2, 7.0)
    case("mix_p4_d3", 3, [(0.0, 1.0)] * 3, [9, 8, 12], ["periodic", "dirichlet", "periodic"], 4, 7.0)

    # FPI (5 iterations) and GMRES through the public drivers on order-4 problems
    g = RH.grid(2, [(0.0, 1.0)] * 2, [24, 24], "periodic")
    f = wh.driver.gaussian_source(g, 6.1, -80.0, 25.0, (0.45, 0.55))
    fpi = {"iter_sha256": [], "residuals": []}
    for k, vk, r in RH.fpi_iterates(g, f, 6.1, 5, p=4):
        fpi["iter_sha256"].append(sha(vk))
        fpi["residuals"].append(float(r))
    cases["fpi_per_p4"] = fpi
    arrays["fpi_per_p4__f"] = np.array(f.values)
    g1 = RH.grid(1, [(0.0, 1.0)], [32], "dirichlet")
    f1 = wh.driver.gaussian_source(g1, 5.5, -100.0, 30.0, 0.37)
    prob = wh.driver.HelmholtzProblem(g1, 4, 1.0, 5.5, f1)
    cfg0 = wh.filters.FilterConfig(omega=5.5, periods=1, steps_per_period=10, mode="explicit")
    x, run = wh.driver.krylov_solve(prob, cfg0, tol=1e-10)
    vf, runf = wh.driver.fpi_solve(prob, cfg0, tol=1e-10, maxit=800)
    cases["gmres_p4_1d"] = {"iterations": run.iterations, "residuals": [float(r) for r in run.residuals],
                            "fpi_iterations": runf.iterations}
    arrays["gmres_p4_1d__x"] = np.array(x.values)
    arrays["gmres_p4_1d__fpi"] = np.array(vf.values)
    arrays["gmres_p4_1d__f"] = np.array(f1.values)
    dump("ext", {"cases": cases}, arrays)


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["small", "ext", "cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--procs", type=int, default=4)
    a = ap.parse_args()
    if a.which == "small":
        run_small()
    elif a.which == "ext":
        run_ext()
    elif a.which == "cfg5":
        run_cfg5(a.procs)
    elif a.which == "cfg4":
        run_cfg4()
    else:
        run_cfg(a.which)


if __name__ == "__main__":
    main()
