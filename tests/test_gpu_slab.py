"""GPU: slab-decomposed solves (several whb contexts owning axis-0 plane ranges,
region-split steps, ghost-plane copies) equal the single-domain reference
iterates bitwise.  Runs all slabs in one process on one GPU (LocalHalo); the
cross-rank driver is covered on CPU by tests/test_slab_gloo.py."""

import numpy as np
import pytest

import paper_2504_03074_b200 as wh
from paper_2504_03074_b200 import _native
from paper_2504_03074_b200.slab import DeviceShard, LocalHalo, exchange_forcing, run_local_solve, slab_ranges
from oracle import native as ON
from oracle import waveholtz_oracle as O

pytestmark = pytest.mark.gpu


def _shards(g, f, sched, nslabs):
    ranges = slab_ranges(g.shape[0], nslabs)
    shards = [DeviceShard(g, r) for r in ranges]
    for sh, (p0, p1) in zip(shards, ranges):
        sh.set_schedule(sched)
        sh.upload(_native.F, np.ascontiguousarray(f[p0:p1]))
        sh.zero(_native.V)
    halo = LocalHalo(shards)
    exchange_forcing(shards, halo)
    return shards, halo


@pytest.mark.parametrize("two_step", [True, False])
@pytest.mark.parametrize("cells,nslabs,omega", [((69, 49), 4, 15.0), ((32, 19, 23), 3, 9.0), ((8, 12, 10), 4, 5.0),
                                                ((64, 64, 64), 2, 20.0), ((40, 31), 5, 7.0), ((24, 20, 36), 3, 6.0)])
def test_local_slabs_match_single_domain_bitwise(gpu_available, monkeypatch, cells, nslabs, omega, two_step):
    """FPI across slabs (one-step schedule: whb_step regions; two-step: whb_pair regions with
    2-plane halos) equals the single-domain iterates; (8, 12, 10) over 4 slabs leaves slabs of
    2-3 planes, so the pair's boundary regions cover whole slabs"""
    if not two_step:
        monkeypatch.setenv("WHB_TB2", "0")
    d = len(cells)
    g = wh.build_grid(d, [(0.0, 1.0)] * d, cells, "dirichlet")
    f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=2)
    corr = wh.correct_explicit(omega, g, 2, 1.0)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    sched = wh.time_schedule(corr, cfg)
    shards, halo = _shards(g, f, sched, nslabs)
    assert all(sh.steps_per_pass == (2 if two_step else 1) for sh in shards)
    iters = 3
    sums = [sum(run_local_solve(shards, halo)) for _ in range(iters)]
    for sh in shards:
        sh.synchronize()
    v = np.concatenate([sh.download(_native.V) for sh in shards], axis=0)
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    vref, rref = ON.fpi(f, g.spacing, sc, iters)
    assert np.array_equal(v, vref), (corr.steps_per_period, two_step)
    np.testing.assert_allclose(np.sqrt(sums) / np.sqrt(g.size), rref, rtol=1e-12)


@pytest.mark.parametrize("cells,nslabs,omega", [((50, 41), 3, 11.0), ((20, 18, 22), 2, 7.5)])
def test_local_slabs_plain_and_matvec_modes(gpu_available, cells, nslabs, omega):
    """PLAIN (W(v, f)) and AV (v - W(v, 0)) outputs of a slab-decomposed two-step solve"""
    d = len(cells)
    g = wh.build_grid(d, [(0.0, 1.0)] * d, cells, "dirichlet")
    f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 2, seed=5)
    v0 = O.zero_dirichlet(np.random.default_rng(3).standard_normal(g.shape) * 1e-2, ["dirichlet"] * d)
    corr = wh.correct_explicit(omega, g, 2, 1.0)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    shards, halo = _shards(g, f, wh.time_schedule(corr, cfg), nslabs)
    for sh, (p0, p1) in zip(shards, slab_ranges(g.shape[0], nslabs)):
        sh.upload(_native.V, np.ascontiguousarray(v0[p0:p1]))
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    run_local_solve(shards, halo, out_mode=_native.OUT_PLAIN)
    out = np.concatenate([sh.ctx.download(_native.OUT) for sh in shards], axis=0)
    assert np.array_equal(out, ON.wave_solve(v0, f, g.spacing, sc))
    run_local_solve(shards, halo, out_mode=_native.OUT_AV, zero_forcing=True)
    out = np.concatenate([sh.ctx.download(_native.OUT) for sh in shards], axis=0)
    assert np.array_equal(out, v0 - ON.wave_solve(v0, f, g.spacing, sc, zero_f=True))


@pytest.mark.parametrize("cells,nslabs,omega", [((60, 44), 3, 9.0), ((24, 20, 26), 4, 7.0)])
def test_slab_krylov_local_matches_single_domain(gpu_available, cells, nslabs, omega):
    """GMRES with the Krylov basis sharded over in-process slabs (ShardedVectors; mat-vecs as
    two-step slab solves) against the single-domain device GMRES and the oracle."""
    from paper_2504_03074_b200.slab import SlabKrylov

    d = len(cells)
    g = wh.build_grid(d, [(0.0, 1.0)] * d, cells, "dirichlet")
    f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=2)
    corr = wh.correct_explicit(omega, g, 2, 1.0)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    ranges = slab_ranges(g.shape[0], nslabs)
    shards = [DeviceShard(g, r) for r in ranges]
    solver = SlabKrylov(shards, LocalHalo(shards), corr, cfg, [f[p0:p1] for p0, p1 in ranges])
    xs, rep = solver.solve(tol=1e-9, restart=8, maxit=40)
    x = np.concatenate(xs, axis=0)
    prob = wh.HelmholtzProblem(g, 2, 1.0, omega, wh.GridField.from_values(g, f))
    xw, run = wh.krylov_solve(prob, cfg, tol=1e-9, restart=8, maxit=40)
    assert rep.iterations == run.iterations
    np.testing.assert_allclose(rep.residual_history, run.residuals, rtol=1e-8)
    assert np.max(np.abs(x - xw.values)) <= 1e-9 * np.max(np.abs(xw.values))
    for sh in shards:
        sh.ctx.close()
