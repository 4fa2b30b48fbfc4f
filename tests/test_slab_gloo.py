"""CPU, world_size 2 (gloo over 127.0.0.1): the slab-decomposition driver
(paper_2504_03074_b200.slab) — plane ranges, halo exchange schedule, residual
all-reduce — run with a numpy stand-in for the device shard, checked bitwise
against the single-domain oracle.  (On the GPU the same driver runs
DeviceShard; tests/test_gpu_slab.py checks the device kernels' region split.)"""

import contextlib
import math
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

from paper_2504_03074_b200 import _native
from paper_2504_03074_b200.grid import build_grid, operator_coefficients
from paper_2504_03074_b200.slab import SlabFPI, TorchHalo, slab_ranges
from paper_2504_03074_b200.timestep import correct_explicit, time_schedule
from paper_2504_03074_b200.filters import FilterConfig
from oracle import native as ON
from oracle import waveholtz_oracle as O
from slab_numpy import NumpyShard, NumpyVecs  # noqa: F401


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dim, cells, omega, iters, q, spp):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = build_grid(dim, [(0.0, 1.0)] * dim, cells, "dirichlet")
        f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=7)
        corr = correct_explicit(omega, g, 2, 1.0)
        cfg = FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
        rng = slab_ranges(g.shape[0], world)[rank]
        shard = NumpyShard(g, rng, steps_per_pass=spp[rank] if isinstance(spp, tuple) else spp)
        solver = SlabFPI(shard, TorchHalo(dist, rank, world), corr, cfg, f)
        res = [solver.iterate() for _ in range(iters)]
        q.put((rank, rng, solver.local_iterate(), res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dim,cells,omega,spp,world", [(2, (40, 24), 12.0, 1, 2), (3, (14, 10, 12), 6.5, 1, 2),
                                                       (2, (40, 24), 12.0, 2, 2), (3, (14, 10, 12), 6.5, 2, 2),
                                                       (3, (14, 10, 12), 6.5, 2, 3), (2, (9, 30), 8.0, 2, 3),
                                                       (3, (20, 10, 12), 6.5, 3, 2), (3, (20, 10, 12), 7.0, 3, 3), (3, (20, 10, 12), 6.75, 3, 2),
                                                       (2, (9, 30), 8.0, 3, 3), (3, (20, 10, 12), 6.5, (3, 2, 3), 3)])
def test_slab_fpi_gloo_matches_single_domain(dim, cells, omega, spp, world):
    """world 2 and 3 (a middle slab exchanges both sides; (9, 30) over 3 ranks leaves
    slabs of 3 and 4 planes, so the two-/three-step boundary regions cover whole slabs).
    spp 3: three-step passes with a 2- or 1-step remainder; (3, 2, 3): ranks whose plans
    differ agree on the smallest (all-reduce MIN) and run two-step passes."""
    iters = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dim, cells, omega, iters, q, spp)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort(key=lambda t: t[0])
    g = build_grid(dim, [(0.0, 1.0)] * dim, cells, "dirichlet")
    v = np.concatenate([t[2] for t in got], axis=0)
    assert [t[1] for t in got] == slab_ranges(g.shape[0], world)
    f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=7)
    corr = correct_explicit(omega, g, 2, 1.0)
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    vref, rref = O.fpi(f, g.spacing, sc, iters)
    assert np.array_equal(v, vref)
    np.testing.assert_allclose(got[0][3], rref, rtol=1e-12)
    assert all(t[3] == got[0][3] for t in got)


@pytest.mark.parametrize("n_total,spp,plan", [
    (10, 3, [(0, 3), (3, 3), (6, 3), (9, 1)]), (11, 3, [(0, 3), (3, 3), (6, 3), (9, 2)]),
    (9, 3, [(0, 3), (3, 3), (6, 3)]), (3, 3, [(0, 2), (2, 1)]), (2, 3, [(0, 2)]),
    (5, 2, [(0, 2), (2, 2), (4, 1)]), (4, 2, [(0, 2), (2, 2)]), (3, 1, [(0, 1), (1, 1), (2, 1)])])
def test_pass_plan_matches_whole_grid_order(n_total, spp, plan):
    """slab.pass_plan orders passes like whb200.cu enqueue_solve (a three-step pass is never both
    the first and the last: n_total <= 3 runs the two-step schedule)."""
    from paper_2504_03074_b200.slab import halo_items, level, pass_plan

    assert pass_plan(n_total, spp) == plan
    assert sum(k for _, k in plan) == n_total
    assert halo_items(0, 3, 3) == [(level(3), 3), (level(2), 2)]
    assert halo_items(3, 3, 1) == [(level(6), 1)]
    assert halo_items(0, 2, 2) == [(level(2), 2), (level(1), 1)]


def test_slab_ranges():
    assert slab_ranges(1025, 8) == [(0, 129)] + [(129 + 128 * i, 257 + 128 * i) for i in range(7)]
    assert [b - a for a, b in slab_ranges(1025, 8)] == [129] + [128] * 7
    assert slab_ranges(10, 1) == [(0, 10)]
    with pytest.raises(ValueError):
        slab_ranges(3, 4)


def _krylov_worker(rank, world, port, cells, omega, q):
    import torch.distributed as dist

    from paper_2504_03074_b200.slab import SlabKrylov

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dim = len(cells)
        g = build_grid(dim, [(0.0, 1.0)] * dim, cells, "dirichlet")
        f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=7)
        corr = correct_explicit(omega, g, 2, 1.0)
        cfg = FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
        p0, p1 = slab_ranges(g.shape[0], world)[rank]
        shard = NumpyShard(g, (p0, p1))
        solver = SlabKrylov([shard], TorchHalo(dist, rank, world), corr, cfg, [f[p0:p1]])
        xs, rep = solver.solve(tol=1e-9, restart=6, maxit=30)
        q.put((rank, xs[0], rep.iterations, rep.residual_history))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cells,omega,world", [((30, 22), 9.0, 2), ((12, 10, 11), 6.5, 3)])
def test_slab_krylov_gloo_matches_single_domain(cells, omega, world):
    """GMRES with the Krylov basis sharded over z-slabs (dots all-reduced across ranks,
    mat-vecs as slab solves with halo exchange) against the single-domain oracle GMRES."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_krylov_worker, args=(r, world, port, cells, omega, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=180) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dim = len(cells)
    g = build_grid(dim, [(0.0, 1.0)] * dim, cells, "dirichlet")
    f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=7)
    corr = correct_explicit(omega, g, 2, 1.0)
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    b = O.wave_solve_filtered(np.zeros(g.shape), f, g.spacing, sc)
    scale = math.sqrt(g.size)
    xref, hist, its, conv = O.gmres(lambda x: O.apply_A(x, g.spacing, sc), b, tol=0.0, restart=6, maxit=30,
                                    atol=1e-9 * scale)
    x = np.concatenate([t[1] for t in got], axis=0)
    assert all(t[2] == its for t in got)
    np.testing.assert_allclose(got[0][3], np.array(hist) / scale, rtol=1e-8)
    assert np.max(np.abs(x - xref)) <= 1e-9 * np.max(np.abs(xref))


def _batch_worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2504_03074_b200.batch as B

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # the device solve replaced by the oracle (host logic under test: sharding + gathers)
        def fake(grid, forcing, omegas, tol=1e-10, maxit=500, c=1.0, order=2, periods=1, device=0):
            from paper_2504_03074_b200.driver import WaveHoltzRun
            from paper_2504_03074_b200.grid import GridField

            out = []
            f = np.asarray(forcing.values)
            for w in omegas:
                corr = correct_explicit(w, grid, order, c)
                sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
                v, res = O.fpi(f, grid.spacing, sc, maxit)
                out.append((GridField.from_values(grid, v), WaveHoltzRun("fpi", periods, list(res), maxit, False)))
            return out

        B.fpi_solve_batched = fake
        g = build_grid(2, [(0.0, 1.0)] * 2, (16, 12), "dirichlet")
        f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 2, seed=3)
        from paper_2504_03074_b200.grid import GridField

        omegas = [4.0, 6.5, 9.0, 11.5, 14.0]
        out = B.fpi_solve_batched_distributed(g, GridField.from_values(g, f), omegas, dist, tol=-1.0, maxit=2,
                                             device=0, gather_iterates=True)
        q.put((rank, [run.residuals for _, run in out], [None if v is None else np.asarray(v.values) for v, _ in out]))
    finally:
        dist.destroy_process_group()


def test_batched_distributed_gathers_runs_world2():
    """config 5 across ranks: LPT sharding of the omegas, runs gathered on every rank, iterates on
    rank 0, each equal to its single-omega solve."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=180) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = build_grid(2, [(0.0, 1.0)] * 2, (16, 12), "dirichlet")
    f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 2, seed=3)
    for k, w in enumerate([4.0, 6.5, 9.0, 11.5, 14.0]):
        corr = correct_explicit(w, g, 2, 1.0)
        sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
        v, res = O.fpi(f, g.spacing, sc, 2)
        assert got[0][1][k] == list(res) and got[1][1][k] == list(res)
        assert np.array_equal(got[0][2][k], v)


def test_nccl_halo_posts_the_torch_halo_pairs():
    """NcclHalo (the C-ABI NCCL path) posts, per item and neighbour, the same (send planes, recv
    planes, peer) as the torch.distributed path, as ONE group between whb_comm_begin / end, and
    joins in finish -- checked with a recording stand-in for the context (world 3, middle rank)."""
    from paper_2504_03074_b200.slab import NcclHalo, halo_planes, level, field

    calls = []

    class Ctx:
        def nccl_init(self, *a):
            calls.append(("init",) + a[:2])

        def comm_begin(self):
            calls.append(("begin",))

        def comm_end(self):
            calls.append(("end",))

        def comm_join(self):
            calls.append(("join",))

        def nccl_exchange(self, *a):
            calls.append(("exchange",) + tuple(list(x) for x in a))

    class Shard:
        gh, nloc = 2, 7
        ctx = Ctx()

        def plane_ptr(self, item, plane):
            base = {level(3): 10_000, level(2): 20_000, field(_native.F): 30_000}[item]
            return base + 100 * plane, 50

    import paper_2504_03074_b200.slab as slab_mod

    old = slab_mod._native.nccl_unique_id
    slab_mod._native.nccl_unique_id = lambda: b"x" * 128
    try:
        sh = Shard()

        class Dist:
            @staticmethod
            def broadcast_object_list(lst, src):
                lst[0] = b"x" * 128

        h = NcclHalo(sh, Dist, 1, 3)
        h.finish(h.start(sh, [(level(3), 2), (level(2), 1)]))
    finally:
        slab_mod._native.nccl_unique_id = old
    assert calls[0] == ("init", 3, 1)
    assert [c[0] for c in calls[1:]] == ["begin", "exchange", "end", "join"]
    _, sends, recvs, counts, peers = calls[2]
    want = []
    for item, depth, base in ((level(3), 2, 10_000), (level(2), 1, 20_000)):
        for q, side in ((0, "lo"), (2, "hi")):
            snd, rcv = halo_planes(sh, side, depth)
            want.append((base + 100 * snd, base + 100 * rcv, 50 * depth, q))
    assert list(zip(sends, recvs, counts, peers)) == want
