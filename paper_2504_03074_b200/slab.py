"""Slab (axis-0) domain decomposition of the explicit WaveHoltz iteration across
GPUs — SURVEY §8(e).

The stencil radius is 1, so every leapfrog step needs exactly one ghost plane
of W^n from each neighbour; W^{n-1}, f and the accumulator are purely local.
Each rank owns a contiguous range of axis-0 planes (``slab_ranges``) in one
whb context (include/whb200.h: plane_begin/plane_end) whose allocation carries
one ghost plane on each side.  Per leapfrog step s:

    1. compute the first and last owned planes of W^{s+1}      (whb_step region 1)
    2. post the halo exchange of those planes                    (NCCL send/recv)
    3. compute the remaining interior planes                     (whb_step region 2)
    4. join the exchange before step s+1                         (stream wait)

so the transfer of 2 x (n1 x n2 x 8 B) per step overlaps the interior update.
Per pass the residual sum of squares is all-reduced (one fp64).

The exchange goes through ``torch.distributed`` (NCCL on GPUs, gloo on CPUs)
on the context's own CUDA stream (``torch.cuda.ExternalStream``); device
buffers are wrapped zero-copy through ``__cuda_array_interface__``.  The
in-process ``LocalHalo`` runs several slabs in one process (one GPU or
several) with device-to-device plane copies, which is how the multi-slab
kernels are checked on a single GPU.
"""

from __future__ import annotations

import contextlib
import math

import numpy as np

from . import _native
from .filters import mode_name
from .grid import operator_coefficients
from .timestep import time_schedule

__all__ = ["slab_ranges", "DeviceShard", "TorchHalo", "LocalHalo", "SlabFPI", "run_filtered_solve"]


def slab_ranges(n0: int, nranks: int):
    """Contiguous, near-equal [p0, p1) ranges of the n0 axis-0 planes (1025 / 8 -> 128 or 129)."""
    if nranks < 1 or nranks > n0:
        raise ValueError("need 1 <= nranks <= number of planes")
    base, extra = divmod(n0, nranks)
    out, p = [], 0
    for r in range(nranks):
        q = p + base + (1 if r < extra else 0)
        out.append((p, q))
        p = q
    return out


class _CudaArray:
    """Minimal __cuda_array_interface__ exporter for a raw device pointer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": (int(n),), "typestr": "<f8",
                                         "strides": None, "version": 3}


class DeviceShard:
    """One rank's slab on its GPU: a whb context owning planes [p0, p1)."""

    def __init__(self, grid, plane_range, c=1.0, order=2, device=0):
        clo, cmid, c2 = operator_coefficients(grid, order, c)
        self.grid = grid
        self.plane_range = tuple(plane_range)
        self.ctx = _native.Context(grid.shape, device=device, plane_range=plane_range)
        self.ctx.set_operator(clo, cmid, c2)
        self.nloc = self.plane_range[1] - self.plane_range[0]
        self.device = device

    # schedule / fields
    def set_schedule(self, sched):
        self.ctx.set_schedule(0, sched)
        self.n_total = sched["n_total"]

    def upload(self, field, local_values):
        self.ctx.upload(field, local_values)

    def download(self, field):
        return self.ctx.download(field)

    def zero(self, field):
        self.ctx.zero(field)

    # step-level control
    def solve_begin(self, out_mode, zero_forcing=False):
        self.ctx.solve_begin(out_mode, zero_forcing)

    def step(self, s, region):
        self.ctx.step(s, region)

    def solve_end(self) -> float:
        return self.ctx.solve_end()

    # halo plumbing
    def plane_tensor(self, level, plane):
        import torch

        ptr, n = self.ctx.level_plane_ptr(level, plane)
        return torch.as_tensor(_CudaArray(ptr, n), device=f"cuda:{self.device}")

    def stream(self):
        import torch

        return torch.cuda.stream(torch.cuda.ExternalStream(self.ctx.stream_ptr(), device=f"cuda:{self.device}"))

    def synchronize(self):
        self.ctx.synchronize()


class TorchHalo:
    """Halo exchange between ranks with torch.distributed point-to-point ops."""

    def __init__(self, dist, rank: int, world: int):
        self.dist = dist
        self.rank = rank
        self.world = world

    @property
    def nranks(self):
        return self.world

    def start(self, shard, level):
        d = self.dist
        ops = []
        with shard.stream():
            if self.rank > 0:
                ops.append(d.P2POp(d.isend, shard.plane_tensor(level, 1), self.rank - 1))
                ops.append(d.P2POp(d.irecv, shard.plane_tensor(level, 0), self.rank - 1))
            if self.rank < self.world - 1:
                ops.append(d.P2POp(d.isend, shard.plane_tensor(level, shard.nloc), self.rank + 1))
                ops.append(d.P2POp(d.irecv, shard.plane_tensor(level, shard.nloc + 1), self.rank + 1))
            works = d.batch_isend_irecv(ops) if ops else []
        return shard, works

    def finish(self, handle):
        shard, works = handle
        with shard.stream():
            for w in works:
                w.wait()

    def allreduce_sum(self, x: float, shard) -> float:
        import torch

        dev = "cpu" if self.dist.get_backend() == "gloo" else f"cuda:{shard.device}"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t)
        return float(t.item())


class LocalHalo:
    """All slabs live in this process: plane copies between contexts (same or peer GPU)."""

    def __init__(self, shards):
        self.shards = list(shards)

    @property
    def nranks(self):
        return len(self.shards)

    def exchange(self, level):
        sh = self.shards
        for r in range(len(sh) - 1):
            lo, hi = sh[r], sh[r + 1]
            lo.ctx.copy_plane_to(level, lo.nloc, hi.ctx, level, 0)
            hi.ctx.copy_plane_to(level, 1, lo.ctx, level, lo.nloc + 1)


def run_filtered_solve(shard, halo, out_mode=_native.OUT_FPI, zero_forcing=False) -> float:
    """One W(v, f) pass of a slab with halo exchange (the step schedule above).
    Returns this rank's residual sum of squares (FPI mode)."""
    shard.solve_begin(out_mode, zero_forcing)
    if halo.nranks > 1:
        halo.finish(halo.start(shard, 0))  # ghost planes of W^0 = v
    n_total = shard.n_total
    for s in range(n_total):
        if halo.nranks == 1 or s == n_total - 1:
            shard.step(s, 0)  # the last step writes the output; no later step needs its halo
            continue
        shard.step(s, 1)
        h = halo.start(shard, s + 1)
        shard.step(s, 2)
        halo.finish(h)
    return shard.solve_end()


def run_local_solve(shards, halo: LocalHalo, out_mode=_native.OUT_FPI, zero_forcing=False):
    """The same schedule for in-process slabs (each step: boundary planes of every slab,
    plane copies, interior planes)."""
    for sh in shards:
        sh.solve_begin(out_mode, zero_forcing)
    halo.exchange(0)
    n_total = shards[0].n_total
    for s in range(n_total):
        if s == n_total - 1:
            for sh in shards:
                sh.step(s, 0)
            continue
        for sh in shards:
            sh.step(s, 1)
        halo.exchange(s + 1)
        for sh in shards:
            sh.step(s, 2)
    return [sh.solve_end() for sh in shards]


class SlabFPI:
    """Fixed-point iteration (driver.py:211-230) over a slab-decomposed grid.

    ``shard`` is this rank's DeviceShard, ``halo`` a TorchHalo.  ``forcing``
    is either the full field (sliced here) or this rank's owned planes.
    """

    def __init__(self, shard, halo, corr, config, forcing):
        if mode_name(config.mode) != "explicit":
            raise NotImplementedError("only the explicit path runs on the GPU")
        self.shard = shard
        self.halo = halo
        self.grid = shard.grid
        shard.set_schedule(time_schedule(corr, config))
        p0, p1 = shard.plane_range
        fv = np.asarray(forcing.values if hasattr(forcing, "values") else forcing, dtype=float)
        if fv.shape[0] == self.grid.shape[0] and fv.shape[0] != p1 - p0:
            fv = fv[p0:p1]
        shard.upload(_native.F, np.ascontiguousarray(fv))
        self.reset()

    def reset(self):
        self.shard.zero(_native.V)

    def iterate(self) -> float:
        """One pass; returns the global scaled residual ||v_new - v||_2 / sqrt(N)."""
        rs = run_filtered_solve(self.shard, self.halo)
        total = self.halo.allreduce_sum(rs, self.shard) if self.halo.nranks > 1 else rs
        return math.sqrt(total) / math.sqrt(self.grid.size)

    def local_iterate(self) -> np.ndarray:
        return self.shard.download(_native.V)
