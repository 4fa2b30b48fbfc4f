"""TEST INFRASTRUCTURE ONLY — drive the real reference package (this container only).

The reference (``/root/reference/pkg/src/waveholtz``) is pure Python/numpy and
importable here; it does NOT exist on the GPU box, so nothing that runs there
may import this module.  It is used by ``tests/golden/make_golden.py`` to
produce the committed golden fixtures and by the CPU test-suite (skipped when
the reference is absent) to pin the numpy/C restatements.

Seams used:
  * ``waveholtz.timestep._COURANT[2]`` — the hard-coded Courant bound
    (timestep.py:43) — set to 0.9 for BASELINE's "CFL 0.9".
  * 3D grids: ``CartesianGrid.__post_init__`` rejects dim=3 (grid.py:66-67);
    everything downstream is dimension generic, so a 3D grid is built with
    ``object.__new__`` + ``object.__setattr__``.
  * per-iterate capture: ``waveholtz.driver`` imports ``wave_solve_filtered``
    by name (driver.py:38) and calls it at driver.py:222/258/280, so rebinding
    ``waveholtz.driver.wave_solve_filtered`` captures every iterate.
"""

from __future__ import annotations

import contextlib
import os
import sys

REFERENCE_SRC = os.environ.get("WHB_REFERENCE_SRC", "/root/reference/pkg/src")


def available() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "waveholtz"))


def import_reference():
    """Import and return the reference ``waveholtz`` package."""
    if not available():
        raise ImportError(f"reference package not found under {REFERENCE_SRC}")
    sys.dont_write_bytecode = True  # the tree is read-only
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import waveholtz  # noqa: F401
    import waveholtz.driver  # noqa: F401
    import waveholtz.timestep  # noqa: F401

    return waveholtz


@contextlib.contextmanager
def courant(value: float, p: int = 2):
    """Temporarily set the reference's Courant bound ``_COURANT[p]`` (timestep.py:43)."""
    wh = import_reference()
    table = wh.timestep._COURANT
    old = table[p]
    table[p] = value
    try:
        yield
    finally:
        table[p] = old


def grid(dim, bounds, cells, bcs="dirichlet"):
    """Reference CartesianGrid; 3D bypasses the dim validator (grid.py:65-74)."""
    wh = import_reference()
    G = wh.grid
    if dim in (1, 2):
        return G.build_grid(dim, bounds, cells, bcs)
    g = object.__new__(G.CartesianGrid)
    per_axis = [bcs] * dim if isinstance(bcs, str) else list(bcs)
    object.__setattr__(g, "dim", dim)
    object.__setattr__(g, "bounds", tuple((float(lo), float(hi)) for lo, hi in bounds))
    object.__setattr__(g, "cells", tuple(int(n) for n in cells))
    object.__setattr__(g, "bcs", tuple(G._as_bc(b) for b in per_axis))
    return g


def multi_gaussian(g, omega, n_gauss, seed=0):
    """BASELINE forcing recipe summed with the reference's gaussian_source.

    rng = default_rng(seed); amp ~ U(-100,100,K); ctr ~ U(0.1,0.9,(K,d));
    b ~ U(100,1000,K); f = sum_k gaussian_source(grid, omega, amp[k], b[k], ctr[k])
    in k order from zeros (driver.py:163-179), then boundary-zeroed.
    """
    import numpy as np

    wh = import_reference()
    rng = np.random.default_rng(seed)
    amp = rng.uniform(-100.0, 100.0, n_gauss)
    ctr = rng.uniform(0.1, 0.9, (n_gauss, g.dim))
    b = rng.uniform(100.0, 1000.0, n_gauss)
    f = np.zeros(g.shape)
    for k in range(n_gauss):
        f = f + wh.driver.gaussian_source(g, omega, amp[k], b[k], ctr[k]).values
    return wh.grid.GridField.from_values(g, f)


def multi_gaussian_slabs(g, omega, n_gauss, seed=0, slab=32):
    """multi_gaussian() for grids too large for the reference's whole-grid numpy
    temporaries (1025^3: ~6 x 8.6 GB per Gaussian): the reference's own
    ``gaussian_source`` (driver.py:163-179) is evaluated on axis-0 slabs of the
    grid through a slab-view grid whose ``coords()`` are the full grid's
    ``axis_coords`` (grid.py:104-112) with axis 0 sliced, so every element goes
    through the same numpy ufuncs on the same operands.  The slab view marks
    axis 0 periodic so ``GridField.from_values`` does not zero the slab's cut
    faces; the global Dirichlet planes 0 and n0-1 are zeroed here exactly as
    ``_enforce_dirichlet_zeros`` (grid.py:237-246) zeroes them on the full grid.
    Returns a plain float64 array of the grid's shape."""
    import numpy as np

    wh = import_reference()
    G = wh.grid
    rng = np.random.default_rng(seed)
    amp = rng.uniform(-100.0, 100.0, n_gauss)
    ctr = rng.uniform(0.1, 0.9, (n_gauss, g.dim))
    b = rng.uniform(100.0, 1000.0, n_gauss)
    shape = tuple(g.shape)
    axes = [g.axis_coords(m) for m in range(g.dim)]
    out = np.empty(shape)

    class _SlabView(G.CartesianGrid):
        def __post_init__(self):
            pass

        @property
        def npoints(self):
            return (self._p1 - self._p0,) + tuple(shape[1:])

        def coords(self):
            ax = [axes[0][self._p0:self._p1]] + axes[1:]
            return tuple(np.meshgrid(*ax, indexing="ij"))

    for p0 in range(0, shape[0], slab):
        p1 = min(shape[0], p0 + slab)
        sv = _SlabView(g.dim, g.bounds, g.cells, (G.BC.PERIODIC,) + tuple(g.bcs[1:]))
        object.__setattr__(sv, "_p0", p0)
        object.__setattr__(sv, "_p1", p1)
        acc = np.zeros(sv.npoints)
        for k in range(n_gauss):
            v = np.array(wh.driver.gaussian_source(sv, omega, amp[k], b[k], ctr[k]).values)
            if p0 == 0:
                v[0] = 0.0
            if p1 == shape[0]:
                v[-1] = 0.0
            acc = acc + v
        if p0 == 0:
            acc[0] = 0.0
        if p1 == shape[0]:
            acc[-1] = 0.0
        out[p0:p1] = acc
    return out


def explicit_setup(g, omega, p=2, c=1.0, periods=1):
    """(corr, cfg, op) exactly as resolve_time_discretization builds them (driver.py:182-192)."""
    wh = import_reference()
    corr = wh.timestep.correct_explicit(omega, g, p, c)
    cfg = wh.filters.FilterConfig(omega=omega, periods=periods,
                                  steps_per_period=corr.steps_per_period, mode="explicit")
    op = wh.grid.DiscreteOperator(g, p, c)
    return corr, cfg, op


def fpi_iterates(g, f_field, omega, iters, p=2, c=1.0, periods=1, callback=None):
    """Run the reference's own _iterate loop body (driver.py:215-230) for exactly
    ``iters`` iterations, yielding (k, v_k ndarray, residual_k).

    Equivalent to ``fpi_solve(prob, cfg, tol=-1.0, maxit=iters)`` with the
    iterate-capturing seam, but does not construct ``HelmholtzProblem`` (whose
    eigen resonance check is 2D-only and O(N log N) in Python tuples).
    """
    import math

    import numpy as np

    wh = import_reference()
    corr, cfg, op = explicit_setup(g, omega, p, c, periods)
    v = wh.grid.GridField.zeros(g, ghost=max(2, op.ghost_width))
    for k in range(1, iters + 1):
        v_new = wh.timestep.wave_solve_filtered(v, f_field, cfg, corr, op)
        diff = np.linalg.norm(v_new.values - v.values) / math.sqrt(g.size)
        v = v_new
        yield k, v.values, diff
