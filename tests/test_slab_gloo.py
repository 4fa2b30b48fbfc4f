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


class NumpyShard:
    """Test double with DeviceShard's interface; arithmetic in reference order
    (the same restatement as oracle/waveholtz_oracle.py, per plane)."""

    def __init__(self, grid, plane_range, c=1.0):
        self.grid = grid
        self.plane_range = tuple(plane_range)
        self.nloc = plane_range[1] - plane_range[0]
        self.clo, self.cmid, self.c2 = operator_coefficients(grid, 2, c)
        shp = (self.nloc + 2,) + tuple(grid.shape[1:])
        self.buf = {k: np.zeros(shp) for k in ("v", "f", "wa", "wb", "acc")}
        self.device = 0
        n0 = grid.shape[0]
        g_lo, g_hi = max(plane_range[0], 1), min(plane_range[1], n0 - 1)
        self.lo, self.hi = g_lo - plane_range[0] + 1, max(g_hi - plane_range[0] + 1, g_lo - plane_range[0] + 1)

    def set_schedule(self, sched):
        self.sc = sched
        self.n_total = sched["n_total"]

    def _field(self, field):
        return {_native.V: "v", _native.F: "f", _native.WA: "wa", _native.WB: "wb", _native.ACC: "acc"}[field]

    def upload(self, field, vals):
        a = np.array(vals, dtype=float)
        for ax in range(1, a.ndim):
            sl = [slice(None)] * a.ndim
            for e in (0, -1):
                sl[ax] = e
                a[tuple(sl)] = 0.0
        if self.plane_range[0] == 0:
            a[0] = 0.0
        if self.plane_range[1] == self.grid.shape[0]:
            a[-1] = 0.0
        self.buf[self._field(field)][1:self.nloc + 1] = a

    def download(self, field):
        return np.array(self.buf[self._field(field)][1:self.nloc + 1])

    def zero(self, field):
        self.buf[self._field(field)][...] = 0.0

    def level(self, L):
        return self.buf["v"] if L == 0 else (self.buf["wa"] if L % 2 else self.buf["wb"])

    def solve_begin(self, out_mode, zero_forcing=False):
        self.mode = out_mode
        self.rs = 0.0

    def _lap(self, w, i):
        lap = 0.0
        lap = lap + self.clo[0] * w[i - 1][..., 1:-1]
        lap = lap + self.cmid[0] * w[i][..., 1:-1]
        lap = lap + self.clo[0] * w[i + 1][..., 1:-1]
        if w.ndim == 3:
            lap = lap[1:-1]
            lap = lap + self.clo[1] * w[i][:-2, 1:-1]
            lap = lap + self.cmid[1] * w[i][1:-1, 1:-1]
            lap = lap + self.clo[1] * w[i][2:, 1:-1]
            c = w[i][1:-1]
        else:
            c = w[i]
        lap = lap + self.clo[-1] * c[..., :-2]
        lap = lap + self.cmid[-1] * c[..., 1:-1]
        lap = lap + self.clo[-1] * c[..., 2:]
        if self.c2 != 1.0:
            lap = lap * self.c2
        return lap

    def step(self, s, region):
        lo, hi = self.lo, self.hi
        planes = {0: range(lo, hi), 1: sorted({lo, hi - 1}) if hi > lo else [], 2: range(lo + 1, hi - 1)}[region]
        sc = self.sc
        w, wp, wn = self.level(s), self.level(s - 1) if s > 0 else None, self.level(s + 1)
        inner = (slice(1, -1),) * (w.ndim - 1)
        for i in planes:
            lap = self._lap(w, i)
            f = self.buf["f"][i][inner]
            wc = w[i][inner]
            if s == 0:
                new = wc + sc["half_dt2"] * (lap - f)
            else:
                new = 2.0 * wc - wp[i][inner] + sc["dt2"] * (lap - f * sc["cos_f"][s])
            acc = self.buf["acc"][i]
            if s == 0:
                acc[inner] = sc["acc_c"][0] * wc
            acc[inner] = acc[inner] + sc["acc_c"][s + 1] * new
            if s == self.n_total - 1:
                out = sc["out_scale"] * acc[inner]
                d = out - self.buf["v"][i][inner]
                self.rs += float(np.sum(d * d))
                self.buf["v"][i][inner] = out
            else:
                wn[i][inner] = new

    def solve_end(self):
        return self.rs

    def plane_tensor(self, level, plane):
        import torch

        return torch.from_numpy(self.level(level)[plane].reshape(-1))

    def stream(self):
        return contextlib.nullcontext()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dim, cells, omega, iters, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = build_grid(dim, [(0.0, 1.0)] * dim, cells, "dirichlet")
        f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=7)
        corr = correct_explicit(omega, g, 2, 1.0)
        cfg = FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
        rng = slab_ranges(g.shape[0], world)[rank]
        shard = NumpyShard(g, rng)
        solver = SlabFPI(shard, TorchHalo(dist, rank, world), corr, cfg, f)
        res = [solver.iterate() for _ in range(iters)]
        q.put((rank, rng, solver.local_iterate(), res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dim,cells,omega", [(2, (40, 24), 12.0), (3, (14, 10, 12), 6.5)])
def test_slab_fpi_world2_gloo_matches_single_domain(dim, cells, omega):
    world, iters = 2, 3
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dim, cells, omega, iters, q)) for r in range(world)]
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
    assert got[0][3] == got[1][3]


def test_slab_ranges():
    assert slab_ranges(1025, 8) == [(0, 129)] + [(129 + 128 * i, 257 + 128 * i) for i in range(7)]
    assert [b - a for a, b in slab_ranges(1025, 8)] == [129] + [128] * 7
    assert slab_ranges(10, 1) == [(0, 10)]
    with pytest.raises(ValueError):
        slab_ranges(3, 4)
