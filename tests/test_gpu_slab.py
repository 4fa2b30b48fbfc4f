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


@pytest.mark.parametrize("cells,nslabs,omega,chunk3,k", [((32, 19, 23), 3, 9.0, 0, 3), ((24, 20, 36), 3, 7.0, 0, 3),
                                                        ((64, 64, 64), 2, 20.0, 9, 3), ((40, 70, 61), 4, 8.0, 4, 3),
                                                        ((8, 12, 10), 4, 5.0, 0, 2), ((30, 13, 17), 1, 6.25, 7, 3)])
def test_local_slabs_three_step_bitwise(gpu_available, monkeypatch, cells, nslabs, omega, chunk3, k):
    """The three-step kernel on slabs (whb_triple regions, 3-plane halos of W^{s+3} + 2 of
    W^{s+2}, f exchanged 2 deep; 2- or 1-step remainder pass) equals the single-domain iterates.
    WHB_T3=1 forces the plan on grids this small; chunk3 > 0 splits region 2 into axis-0 chunks.
    (8, 12, 10) over 4 slabs leaves slabs of 2 planes: the slabs agree on two-step passes."""
    monkeypatch.setenv("WHB_T3", "1")
    if chunk3:
        monkeypatch.setenv("WHB_CHUNK3", str(chunk3))
    d = len(cells)
    g = wh.build_grid(d, [(0.0, 1.0)] * d, cells, "dirichlet")
    f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=2)
    corr = wh.correct_explicit(omega, g, 2, 1.0)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    shards, halo = _shards(g, f, wh.time_schedule(corr, cfg), nslabs)
    assert all(sh.steps_per_pass == 3 for sh in shards)
    assert all(sh.pass_steps == k for sh in shards)
    iters = 3
    sums = [sum(run_local_solve(shards, halo)) for _ in range(iters)]
    for sh in shards:
        sh.synchronize()
    v = np.concatenate([sh.download(_native.V) for sh in shards], axis=0)
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    vref, rref = ON.fpi(f, g.spacing, sc, iters)
    assert np.array_equal(v, vref), (corr.steps_per_period, k)
    np.testing.assert_allclose(np.sqrt(sums) / np.sqrt(g.size), rref, rtol=1e-12)
    # PLAIN and AV outputs through the same three-step slab schedule
    v0 = O.zero_dirichlet(np.random.default_rng(3).standard_normal(g.shape) * 1e-2, ["dirichlet"] * d)
    for sh, (p0, p1) in zip(shards, slab_ranges(g.shape[0], nslabs)):
        sh.upload(_native.V, np.ascontiguousarray(v0[p0:p1]))
    run_local_solve(shards, halo, _native.OUT_PLAIN)
    w = np.concatenate([sh.download(_native.OUT) for sh in shards], axis=0)
    assert np.array_equal(w, ON.wave_solve(v0, f, g.spacing, sc))
    run_local_solve(shards, halo, _native.OUT_AV, zero_forcing=True)
    av = np.concatenate([sh.download(_native.OUT) for sh in shards], axis=0)
    assert np.array_equal(av, v0 - ON.wave_solve(v0, f, g.spacing, sc, zero_f=True))


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


@pytest.mark.parametrize("two_step", [True, False])
@pytest.mark.parametrize("cells,nslabs,omega", [((69, 49), 4, 15.0), ((32, 19, 23), 3, 9.0), ((8, 12, 10), 4, 5.0),
                                                ((64, 64, 64), 2, 20.0)])
def test_peer_halo_slabs_match_single_domain_bitwise(gpu_available, monkeypatch, cells, nslabs, omega, two_step):
    """The peer-memory exchange (slab.PeerHalo): boundary planes copied straight into the
    neighbours' ghost planes on each slab's own stream, ordered by stream flag writes / waits
    between the slabs' streams (no host synchronisation inside a solve)."""
    from paper_2504_03074_b200.slab import PeerHalo, run_peer_local_solve

    if not two_step:
        monkeypatch.setenv("WHB_TB2", "0")
    d = len(cells)
    g = wh.build_grid(d, [(0.0, 1.0)] * d, cells, "dirichlet")
    f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=2)
    corr = wh.correct_explicit(omega, g, 2, 1.0)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    ranges = slab_ranges(g.shape[0], nslabs)
    shards = [DeviceShard(g, r) for r in ranges]
    for sh, (p0, p1) in zip(shards, ranges):
        sh.set_schedule(wh.time_schedule(corr, cfg))
        sh.upload(_native.F, np.ascontiguousarray(f[p0:p1]))
        sh.zero(_native.V)
    halos = PeerHalo.local_group(shards)
    exchange_forcing(shards, halos)
    iters = 3
    sums = [sum(run_peer_local_solve(shards, halos)) for _ in range(iters)]
    v = np.concatenate([sh.download(_native.V) for sh in shards], axis=0)
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    vref, rref = ON.fpi(f, g.spacing, sc, iters)
    assert np.array_equal(v, vref), (corr.steps_per_period, two_step)
    np.testing.assert_allclose(np.sqrt(sums) / np.sqrt(g.size), rref, rtol=1e-12)
    for h in halos:
        h.close()


def _ipc_worker(rank, port, q):
    """Two processes on one GPU: each maps the other's level buffer and flags through CUDA IPC
    (PeerHalo.from_dist), copies its boundary plane into the other's ghost plane and bumps the
    other's flag with a stream write; the host (gloo barrier), not the device, waits."""
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2504_03074_b200.slab import PeerHalo, level

        g = wh.build_grid(2, [(0.0, 1.0)] * 2, [20, 16], "dirichlet")
        sh = DeviceShard(g, slab_ranges(g.shape[0], 2)[rank])
        vals = np.full((sh.nloc, g.shape[1]), float(rank + 1))
        sh.upload(_native.V, vals)
        h = PeerHalo.from_dist(sh, dist, rank, 2)
        seq = h.start(sh, [(level(0), 1)])
        sh.synchronize()
        dist.barrier()
        import torch

        from paper_2504_03074_b200.slab import _CudaArray

        ghost_ptr, n = sh.plane_ptr(level(0), sh.gh - 1 if rank == 1 else sh.gh + sh.nloc)
        got = torch.as_tensor(_CudaArray(ghost_ptr, n), device="cuda").cpu().numpy()
        # the two uint32 flags, read through a one-element float64 view
        raw = torch.as_tensor(_CudaArray(h.flags, 1), device="cuda").cpu().numpy().view(np.uint32)
        dist.barrier()
        h.close()
        q.put((rank, seq, got.tolist(), raw.tolist(), None))
    finally:
        dist.destroy_process_group()


def test_peer_halo_ipc_two_processes(gpu_available):
    import multiprocessing as mp
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=300) for _ in range(2)])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, seq, ghost, flags, _ in got:
        other = 2 - rank  # the neighbour's value (rank 0 holds 1.0, rank 1 holds 2.0)
        g = np.array(ghost)
        # interior columns of the received plane carry the neighbour's value (boundary columns 0)
        assert np.all(g[1:16] == float(other)), (rank, g[:20])
        slot = 1 if rank == 0 else 0  # rank 0 hears from its upper neighbour, rank 1 from its lower one
        assert flags[slot] == seq == 1 and flags[1 - slot] == 0


@pytest.mark.parametrize("cells,nslabs,omega", [((69, 49), 4, 15.0), ((32, 19, 23), 3, 9.0)])
def test_peer_slab_graphs_match_single_domain_bitwise(gpu_available, cells, nslabs, omega):
    """One CUDA graph per slab iteration (kernels + peer copies + stream flag writes / waits),
    replayed: every iterate equals the single-domain reference iterate."""
    from paper_2504_03074_b200.slab import PeerHalo, PeerSlabGraphs

    d = len(cells)
    g = wh.build_grid(d, [(0.0, 1.0)] * d, cells, "dirichlet")
    f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=2)
    corr = wh.correct_explicit(omega, g, 2, 1.0)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    ranges = slab_ranges(g.shape[0], nslabs)
    shards = [DeviceShard(g, r) for r in ranges]
    for sh, (p0, p1) in zip(shards, ranges):
        sh.set_schedule(wh.time_schedule(corr, cfg))
        sh.upload(_native.F, np.ascontiguousarray(f[p0:p1]))
        sh.zero(_native.V)
    halos = PeerHalo.local_group(shards)
    exchange_forcing(shards, halos)
    for h, sh in zip(halos, shards):
        h.epoch_end(sh)
    pg = PeerSlabGraphs(shards, halos)  # the warm-up inside is iterate 1
    sums = [sum(pg.iterate()) for _ in range(3)]
    v = np.concatenate([sh.download(_native.V) for sh in shards], axis=0)
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    vref, rref = ON.fpi(f, g.spacing, sc, 4)
    assert np.array_equal(v, vref)
    np.testing.assert_allclose(np.sqrt(sums) / np.sqrt(g.size), rref[1:], rtol=1e-12)
    for h in halos:
        h.close()


def test_nccl_exchange_in_the_c_abi_self_peer_and_graph(gpu_available):
    """The C-ABI NCCL path on one GPU: a one-rank communicator whose exchange sends two owned
    planes to itself (peer = own rank) into the ghost planes, on the exchange stream between
    whb_comm_begin / whb_comm_end, joined by whb_comm_join -- eagerly and replayed from a captured
    CUDA graph; the ghost planes then hold the owned planes' bits."""
    import paper_2504_03074_b200 as wh
    from paper_2504_03074_b200 import _native
    from paper_2504_03074_b200.slab import DeviceShard, level

    g = wh.build_grid(3, [(0.0, 1.0)] * 3, (20, 18, 22), "dirichlet")
    sh = DeviceShard(g, (0, g.shape[0]))
    ctx = sh.ctx
    ctx.nccl_init(1, 0, _native.nccl_unique_id())
    rng = np.random.default_rng(4)
    gh, n = sh.gh, sh.nloc

    def once():
        sp, cnt = sh.plane_ptr(level(0), gh + 3)
        rp, _ = sh.plane_ptr(level(0), gh - 2)
        ctx.comm_begin()
        ctx.nccl_exchange([sp], [rp], [2 * cnt], [0])
        ctx.comm_end()
        ctx.comm_join()

    for mode in ("eager", "graph"):
        v = rng.standard_normal(g.shape)
        sh.upload(_native.V, v)
        ctx.synchronize()
        if mode == "eager":
            once()
        else:
            ctx.capture_begin()
            once()
            gid = ctx.capture_end()
            ctx.graph_launch(gid)
        ctx.synchronize()
        ghost = sh.planes(level(0), gh - 2, 2).cpu().numpy()
        own = sh.planes(level(0), gh + 3, 2).cpu().numpy()
        assert np.array_equal(ghost, own) and np.any(own != 0.0), mode
    assert ctx.nccl_allreduce_sum(2.5) == 2.5
    ctx.close()
