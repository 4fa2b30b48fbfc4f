"""Batched-frequency WaveHoltz (BASELINE config 5): many independent omegas on
one grid, solved simultaneously.

The reference solves one frequency per call (``fpi_solve``, driver.py:201);
a sweep is a Python loop over omegas.  Here all members share
one grid and one forcing array in HBM, each member carries its own v, leapfrog
pair, accumulator and per-step schedule (its own N_t, dt, omega_e, alpha_d),
and every leapfrog step is ONE kernel launch over all still-active members
(members sorted by N_t, descending, so the active set is a prefix; members
taking their last step get the last-step variant in a second launch).

Across GPUs the members are sharded by longest-processing-time first over
sum(N_t) (``lpt_shard``): the units are independent, there is no data-path
collective.
"""

from __future__ import annotations

import math
import time

import numpy as np

from . import _native
from .filters import FilterConfig
from .grid import GridField, operator_coefficients
from .timestep import correct_explicit, time_schedule

__all__ = ["BatchedFPI", "fpi_solve_batched", "fpi_solve_batched_distributed", "lpt_shard"]


def lpt_shard(weights, nranks: int):
    """Greedy longest-processing-time assignment of items (weights = N_t) to ranks.
    Returns a list of index lists, one per rank (deterministic)."""
    order = sorted(range(len(weights)), key=lambda i: (-weights[i], i))
    loads = [0] * nranks
    out = [[] for _ in range(nranks)]
    for i in order:
        r = min(range(nranks), key=lambda q: (loads[q], q))
        out[r].append(i)
        loads[r] += weights[i]
    return [sorted(x) for x in out]


class BatchedFPI:
    """Device-resident fixed-point iteration for a batch of frequencies on one grid."""

    def __init__(self, grid, forcing, omegas, c: float = 1.0, order: int = 2, periods: int = 1, device: int = 0):
        self.grid = grid
        self.omegas = [float(w) for w in omegas]
        if not self.omegas:
            raise ValueError("need at least one omega")
        self.c = float(c)
        self.corrs = [correct_explicit(w, grid, order, c) for w in self.omegas]
        self.configs = [FilterConfig(omega=w, periods=periods, steps_per_period=k.steps_per_period, mode="explicit")
                        for w, k in zip(self.omegas, self.corrs)]
        clo, cmid, c2 = operator_coefficients(grid, order, c)
        self.ctx = _native.Context(grid.shape, device=device, nbatch=len(self.omegas), shared_forcing=True)
        self.ctx.set_operator(clo, cmid, c2)
        for b, (k, cfg) in enumerate(zip(self.corrs, self.configs)):
            self.ctx.set_schedule(b, time_schedule(k, cfg))
        fv = forcing.values if hasattr(forcing, "values") else np.asarray(forcing, dtype=float)
        self.ctx.upload(_native.F, fv, 0)
        self.reset()

    @property
    def steps(self):
        return [cfg.periods * k.steps_per_period for k, cfg in zip(self.corrs, self.configs)]

    @property
    def updates_per_iteration(self) -> int:
        return int(np.prod(self.grid.shape)) * sum(self.steps)

    def reset(self):
        for b in range(len(self.omegas)):
            self.ctx.zero(_native.V, b)

    def run(self, iters: int) -> np.ndarray:
        """`iters` passes for every member, no host sync in between; returns the
        scaled residuals ||v_{k+1}-v_k||/sqrt(N), shape (iters, B)."""
        rs = self.ctx.fpi(iters)
        return np.sqrt(rs) / math.sqrt(self.grid.size)

    def iterate(self, b: int) -> np.ndarray:
        return self.ctx.download(_native.V, b)

    def close(self):
        self.ctx.close()


def fpi_solve_batched(grid, forcing, omegas, tol=1e-10, maxit=500, c=1.0, order=2, periods=1, device=0):
    """``fpi_solve`` (driver.py:201-244) for every omega at once.

    Each member stops exactly like the reference's loop (first iteration with
    residual <= tol); its returned iterate is the one at that iteration.
    Returns a list of (GridField, dict(residuals, iterations, converged, omega)).
    """
    from .driver import WaveHoltzRun

    solver = BatchedFPI(grid, forcing, omegas, c=c, order=order, periods=periods, device=device)
    B = len(solver.omegas)
    hist = [[] for _ in range(B)]
    done = [None] * B
    t0 = time.perf_counter()
    if tol < 0:
        r = solver.run(maxit)
        for b in range(B):
            hist[b] = list(r[:, b])
    else:
        for _ in range(maxit):
            r = solver.run(1)[0]
            for b in range(B):
                if done[b] is None:
                    hist[b].append(float(r[b]))
                    if r[b] <= tol:
                        done[b] = GridField.from_values(grid, solver.iterate(b))
            if all(d is not None for d in done):
                break
    wall = time.perf_counter() - t0
    out = []
    for b in range(B):
        v = done[b] if done[b] is not None else GridField.from_values(grid, solver.iterate(b))
        run = WaveHoltzRun(method="fpi", periods=periods, residuals=hist[b], iterations=len(hist[b]),
                           converged=done[b] is not None, wall_time=wall)
        out.append((v, run))
    solver.close()
    return out


def fpi_solve_batched_distributed(grid, forcing, omegas, dist, tol=1e-10, maxit=500, c=1.0, order=2, periods=1,
                                  device=None, gather_iterates=False):
    """``fpi_solve_batched`` across the ranks of a ``torch.distributed`` group (one GPU per
    rank): the omegas are LPT-sharded over their N_t (``lpt_shard``), every rank solves its
    share as one batch on its own GPU (no data-path collective), and the only collective is
    the final gather of the runs (residual histories) — SURVEY §8(e), config 5.

    Returns, on every rank, a list over ALL omegas (input order) of
    (GridField or None, WaveHoltzRun): the iterate is present for this rank's own omegas, and
    for every omega when ``gather_iterates`` (rank 0 receives them; other ranks get None)."""
    import os

    rank, world = dist.get_rank(), dist.get_world_size()
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    omegas = [float(w) for w in omegas]
    nts = [correct_explicit(w, grid, order, c).steps_per_period * periods for w in omegas]
    mine = lpt_shard(nts, world)[rank]
    local = fpi_solve_batched(grid, forcing, [omegas[i] for i in mine], tol=tol, maxit=maxit, c=c, order=order,
                              periods=periods, device=device) if mine else []
    runs = {i: run for i, (_, run) in zip(mine, local)}
    parts = [None] * world
    dist.all_gather_object(parts, runs)
    all_runs = {}
    for p in parts:
        all_runs.update(p)
    fields = {i: v for i, (v, _) in zip(mine, local)}
    if gather_iterates:
        payload = {i: np.asarray(v.values) for i, v in fields.items()}
        got = [None] * world if rank == 0 else None
        dist.gather_object(payload, got, dst=0)
        if rank == 0:
            fields = {}
            for part in got:
                fields.update({i: GridField.from_values(grid, a) for i, a in part.items()})
    return [(fields.get(i), all_runs[i]) for i in range(len(omegas))]
