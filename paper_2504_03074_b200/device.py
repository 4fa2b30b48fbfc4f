"""Device-resident problem state: one whb context per (grid, wave speed, device).

The reference re-creates every array per call (timestep.py:282-301).  Here a
grid's device buffers (v, f, leapfrog pair, accumulator) are allocated once
and reused across calls; the forcing is uploaded only when its values change,
and the per-step schedule only when the time correction changes.
"""

from __future__ import annotations

import collections

import numpy as np

from . import _native
from .grid import general_operator, is_fast_operator, operator_coefficients

__all__ = ["DeviceProblem", "device_problem", "release_device_cache"]

_MAX_CACHED = 2
_cache: "collections.OrderedDict[tuple, DeviceProblem]" = collections.OrderedDict()


def set_device_operator(ctx, grid, order, c):
    """p = 2 all-Dirichlet -> the temporal-blocked kernels; anything else (p = 4, periodic or
    mixed boundaries) -> the general one-step kernel."""
    if is_fast_operator(grid, order):
        ctx.set_operator(*operator_coefficients(grid, order, c))
    else:
        ctx.set_operator_general(*general_operator(grid, order, c))


def _grid_key(grid, c, device, nbatch=1, shared=False, order=2):
    return (tuple(int(n) for n in grid.shape), tuple(float(d) for d in grid.spacing), float(c), int(device),
            int(nbatch), bool(shared), int(order))


class DeviceProblem:
    """A grid on one GPU (optionally a batch of problems sharing the grid)."""

    def __init__(self, grid, c=1.0, order=2, device=0, nbatch=1, shared_forcing=False, plane_range=None):
        self.grid = grid
        self.c = float(c)
        self.nbatch = nbatch
        self.ctx = _native.Context(grid.shape, device=device, plane_range=plane_range, nbatch=nbatch,
                                   shared_forcing=shared_forcing)
        set_device_operator(self.ctx, grid, order, c)
        self._sched = [None] * nbatch
        self._forcing = [None] * (1 if shared_forcing else nbatch)
        self._forcing_key = {}
        self.shared_forcing = shared_forcing

    @property
    def npoints(self) -> int:
        return int(np.prod(self.grid.shape))

    def set_schedule(self, sched: dict, member: int = 0):
        key = (sched["n_total"], sched["half_dt2"], sched["dt2"], sched["out_scale"],
               np.asarray(sched["cos_f"]).tobytes(), np.asarray(sched["acc_c"]).tobytes())
        if self._sched[member] != key:
            self.ctx.set_schedule(member, sched)
            self._sched[member] = key

    def set_forcing_field(self, field, member: int = 0) -> bool:
        """set_forcing() for a GridField (ours or the reference's): the device copy is keyed on
        the field object and its write counter (``generation``, grid.py:185-216: values are a
        read-only view, every write goes through set_values / _touch), so an unchanged forcing
        costs no host pass over its values; the cache holds the field, so its id cannot be
        reused while it is keyed.  Returns True when f is identically zero."""
        gen = getattr(field, "generation", None)
        if gen is None:
            return self.set_forcing(field.values, member)
        slot = 0 if self.shared_forcing else member
        key = (id(field), gen)
        cached = self._forcing_key.get(slot)
        if cached is not None and cached[0] == key and cached[1] is field:
            return cached[2]
        vals = field.values
        self.ctx.upload_view(_native.F, vals, member)
        zero = not np.any(vals)  # once per upload (exact: a dot product could underflow to 0)
        self._forcing[slot] = None  # the array-keyed cache no longer describes the device copy
        self._forcing_key[slot] = (key, field, zero)
        return zero

    def set_forcing(self, values, member: int = 0) -> bool:
        """Upload f unless the device already holds exactly these values; returns
        True when f is identically zero (the zero-forcing kernel variant applies)."""
        slot = 0 if self.shared_forcing else member
        vals = np.asarray(values, dtype=np.float64)
        cached = self._forcing[slot]
        if cached is None or cached.shape != vals.shape or not np.array_equal(cached, vals):
            self.ctx.upload(_native.F, vals, member)
            self._forcing[slot] = np.array(vals)
            self._forcing_key.pop(slot, None)
        return not np.any(self._forcing[slot])

    def close(self):
        self.ctx.close()

    def __del__(self):
        try:
            self.ctx.close()
        except Exception:
            pass


def device_problem(grid, c=1.0, order=2, device=0) -> DeviceProblem:
    """Cached single-problem device state for a grid (LRU of a few entries)."""
    key = _grid_key(grid, c, device, order=order) + tuple(str(getattr(b, "value", b)) for b in grid.bcs)
    dp = _cache.get(key)
    if dp is not None:
        _cache.move_to_end(key)
        return dp
    while len(_cache) >= _MAX_CACHED:
        # evicted, not closed: holders (HostFPIStep, waveholtz_operator closures, implicit
        # solvers) may still use it; its device memory is freed when the last reference goes
        _cache.popitem(last=False)
    dp = DeviceProblem(grid, c=c, order=order, device=device)
    _cache[key] = dp
    return dp


def release_device_cache():
    """Free every cached device problem (returns HBM to the allocator)."""
    while _cache:
        _cache.popitem(last=False)
    import gc

    gc.collect()  # contexts nobody else references are freed now (DeviceProblem.__del__)
