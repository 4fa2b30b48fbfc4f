"""Grids, fields and the discrete operator descriptor — host-side mirror of
waveholtz/grid.py (reference file:line cited per item).

These are plain host objects: they carry geometry and field values and hand
the GPU path the exact scalars it needs.  Differences from the reference:
  * ``dim`` may be 1, 2 or 3 (the reference validator allows 1-2,
    grid.py:66-67; its numerics are dimension generic).
  * ``GridField`` stores the stored-point values only; the ghost layer the
    reference keeps for its numpy stencil (grid.py:195-205) is meaningless
    here because the device kernels read neighbours directly.  ``ghost`` is
    kept as an attribute for signature compatibility.
Reference objects (``waveholtz.grid.CartesianGrid`` etc.) are accepted
wherever these are, by duck typing.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

__all__ = [
    "BC", "CartesianGrid", "GridField", "DiscreteOperator", "build_grid", "stencil_coefficients",
    "bc_name", "operator_coefficients", "general_operator", "is_fast_operator",
]


class BC(Enum):
    """grid.py:36-38."""

    DIRICHLET = "dirichlet"
    PERIODIC = "periodic"


def bc_name(bc) -> str:
    """Name of a boundary condition from this package's or the reference's BC enum."""
    return str(getattr(bc, "value", bc)).lower()


def _as_bc(value) -> BC:
    try:
        return BC(bc_name(value))
    except ValueError:
        raise ValueError(f"unknown boundary condition {value!r}") from None


@dataclass(frozen=True)
class CartesianGrid:
    """Tensor-product grid (grid.py:50-137); Dirichlet axes store cells+1 points."""

    dim: int
    bounds: tuple
    cells: tuple
    bcs: tuple

    def __post_init__(self):
        if self.dim not in (1, 2, 3):
            raise ValueError("only 1D, 2D and 3D grids are supported")
        if len(self.bounds) != self.dim or len(self.cells) != self.dim or len(self.bcs) != self.dim:
            raise ValueError("bounds/cells/bcs must have one entry per axis")
        for (lo, hi), n in zip(self.bounds, self.cells):
            if not hi > lo:
                raise ValueError(f"inverted or empty bounds ({lo}, {hi})")
            if n < 4:
                raise ValueError("need at least 4 cells per axis for the stencil")

    @property
    def spacing(self) -> tuple:
        return tuple((hi - lo) / n for (lo, hi), n in zip(self.bounds, self.cells))

    @property
    def lengths(self) -> tuple:
        return tuple(hi - lo for lo, hi in self.bounds)

    @property
    def npoints(self) -> tuple:
        return tuple(n + 1 if bc is BC.DIRICHLET else n for n, bc in zip(self.cells, self.bcs))

    @property
    def shape(self) -> tuple:
        return self.npoints

    @property
    def size(self) -> int:
        return int(np.prod(self.npoints))

    @property
    def cell_volume(self) -> float:
        return float(np.prod(self.spacing))

    def axis_coords(self, axis: int) -> np.ndarray:
        lo = self.bounds[axis][0]
        return lo + self.spacing[axis] * np.arange(self.npoints[axis])

    def coords(self) -> tuple:
        """Coordinates broadcast to the field shape, 'ij' indexing (grid.py:109-112)."""
        axes = [self.axis_coords(m) for m in range(self.dim)]
        return tuple(np.meshgrid(*axes, indexing="ij")) if self.dim > 1 else (axes[0],)

    def interior_slices(self) -> tuple:
        return tuple(slice(1, -1) if bc is BC.DIRICHLET else slice(None) for bc in self.bcs)

    def boundary_mask(self) -> np.ndarray:
        mask = np.zeros(self.shape, dtype=bool)
        for axis, bc in enumerate(self.bcs):
            if bc is BC.DIRICHLET:
                sel = [slice(None)] * self.dim
                for edge in (0, -1):
                    sel[axis] = edge
                    mask[tuple(sel)] = True
        return mask

    @property
    def all_dirichlet(self) -> bool:
        return all(bc is BC.DIRICHLET for bc in self.bcs)

    @property
    def all_periodic(self) -> bool:
        return all(bc is BC.PERIODIC for bc in self.bcs)


def build_grid(dim, bounds, cells, bcs) -> CartesianGrid:
    """Loosely typed constructor with the reference's argument rules (grid.py:140-182)."""
    if hasattr(bounds[0], "__len__"):
        b = tuple((float(p[0]), float(p[1])) for p in bounds)
    elif dim == 1:
        b = ((float(bounds[0]), float(bounds[1])),)
    else:
        raise ValueError(f"{dim}D grids need one (lo, hi) pair per axis")
    if len(b) != dim:
        raise ValueError(f"expected {dim} bound pairs, got {len(b)}")
    c = (int(cells),) * dim if np.isscalar(cells) else tuple(int(n) for n in cells)
    if len(c) != dim:
        raise ValueError(f"expected {dim} cell counts, got {len(c)}")
    if isinstance(bcs, (str, BC)):
        pairs = [(_as_bc(bcs), _as_bc(bcs))] * dim
    else:
        pairs = []
        for e in bcs:
            pairs.append((_as_bc(e), _as_bc(e)) if isinstance(e, (str, BC)) else (_as_bc(e[0]), _as_bc(e[1])))
    if len(pairs) != dim:
        raise ValueError(f"expected {dim} boundary conditions, got {len(pairs)}")
    axis_bcs = []
    for lo, hi in pairs:
        if (lo is BC.PERIODIC) != (hi is BC.PERIODIC):
            raise ValueError("periodic faces must come in matched pairs per axis")
        axis_bcs.append(lo)
    return CartesianGrid(dim=dim, bounds=b, cells=c, bcs=tuple(axis_bcs))


def _zero_dirichlet(grid, arr: np.ndarray) -> np.ndarray:
    """grid.py:237-246 / 395-402."""
    for axis, bc in enumerate(grid.bcs):
        if bc_name(bc) == "dirichlet":
            sel = [slice(None)] * arr.ndim
            for edge in (0, -1):
                sel[axis] = edge
                arr[tuple(sel)] = 0.0
    return arr


class GridField:
    """Stored-point values of a field (grid.py:185-291 contract: read-only ``values``,
    ``set_values`` copies and zeroes Dirichlet points, ``generation`` counts writes)."""

    def __init__(self, grid, ghost: int = 2, values=None):
        if ghost < 1:
            raise ValueError("ghost layer width must be at least 1")
        self.grid = grid
        self.ghost = int(ghost)
        self._vals = np.zeros(tuple(grid.shape), dtype=float)
        self.generation = 0
        if values is not None:
            self.set_values(values)

    @property
    def values(self) -> np.ndarray:
        v = self._vals.view()
        v.flags.writeable = False
        return v

    def set_values(self, arr) -> "GridField":
        a = np.asarray(arr, dtype=float)
        if a.shape != tuple(self.grid.shape):
            raise ValueError(f"shape {a.shape} does not match grid {tuple(self.grid.shape)}")
        self._vals[...] = a
        _zero_dirichlet(self.grid, self._vals)
        self.generation += 1
        return self

    def _writable(self) -> np.ndarray:
        return self._vals

    def _touch(self):
        self.generation += 1

    def copy(self) -> "GridField":
        return GridField(self.grid, self.ghost, self._vals)

    def norm_2h(self) -> float:
        return float(np.linalg.norm(self._vals) / np.sqrt(self.grid.size))

    def dot_volume(self, other) -> float:
        return float(self.grid.cell_volume * np.vdot(self._vals, other.values))

    @classmethod
    def zeros(cls, grid, ghost: int = 2) -> "GridField":
        return cls(grid, ghost)

    @classmethod
    def from_values(cls, grid, arr, ghost: int = 2) -> "GridField":
        return cls(grid, ghost, values=arr)


_TAPS = {2: np.array([1.0, -2.0, 1.0]), 4: np.array([-1.0, 16.0, -30.0, 16.0, -1.0]) / 12.0}


def stencil_coefficients(p: int, dx: float) -> np.ndarray:
    """Central second-difference taps of order p over dx^2 (grid.py:296-306)."""
    if p == 2:
        return np.array([1.0, -2.0, 1.0]) / dx**2
    if p == 4:
        return np.array([-1.0 / 12.0, 4.0 / 3.0, -5.0 / 2.0, 4.0 / 3.0, -1.0 / 12.0]) / dx**2
    raise ValueError(f"unsupported order p={p}; expected 2 or 4")


@dataclass(frozen=True)
class DiscreteOperator:
    """c^2 * order-p Laplacian descriptor (grid.py:309-331); applied on the device."""

    grid: object
    order: int
    c: float = 1.0

    def __post_init__(self):
        if self.order not in (2, 4):
            raise ValueError(f"unsupported order p={self.order}; expected 2 or 4")
        if not self.c > 0:
            raise ValueError("wave speed c must be positive")

    @property
    def ghost_width(self) -> int:
        return self.order // 2

    def stencil(self, axis: int) -> np.ndarray:
        return stencil_coefficients(self.order, self.grid.spacing[axis])

    def apply_values(self, values: np.ndarray, ghost_scratch=None) -> np.ndarray:
        """c^2 * L_h on a stored-point array, Dirichlet rows zero (grid.py:346-352), on the GPU."""
        from . import _native
        from .device import device_problem

        dp = device_problem(self.grid, c=self.c, order=self.order)
        dp.ctx.vec_upload(_native.WA, np.asarray(values, dtype=float))
        dp.ctx.zero(_native.OUT)
        dp.ctx.apply_operator(_native.WA, _native.OUT)
        return dp.ctx.download(_native.OUT)

    def apply(self, u) -> "GridField":
        """grid.py:333-344."""
        if u.grid is not self.grid and u.grid != self.grid:
            raise ValueError("field grid does not match operator grid")
        return GridField(self.grid, u.ghost, self.apply_values(u.values))


def is_fast_operator(grid, order: int) -> bool:
    """p = 2 with homogeneous Dirichlet on every axis: the temporal-blocked kernels apply."""
    return order == 2 and all(bc_name(b) == "dirichlet" for b in grid.bcs)


def general_operator(grid, order: int, c: float):
    """(order, periodic[d], taps[d][p+1], c2) exactly as the reference forms them:
    ``stencil_coefficients(p, dx)`` per axis (grid.py:296-306) and ``c**2`` (grid.py:366).
    Any order in {2, 4} and per-axis Dirichlet / periodic boundaries."""
    if order not in (2, 4):
        raise ValueError(f"unsupported order p={order}; expected 2 or 4")
    periodic = [1 if bc_name(b) == "periodic" else 0 for b in grid.bcs]
    taps = np.array([stencil_coefficients(order, dx) for dx in grid.spacing])
    return order, periodic, taps, float(c**2)


def operator_coefficients(grid, order: int, c: float):
    """(clo[d], cmid[d], c2) exactly as the reference forms them: the taps
    ``np.array([1,-2,1]) / dx**2`` of each axis (grid.py:302-306) and ``c**2``
    (grid.py:366).  Only p = 2 with all-Dirichlet boundaries runs on the GPU."""
    if not is_fast_operator(grid, order):
        raise NotImplementedError("operator_coefficients covers p = 2 / all-Dirichlet; use general_operator")
    taps = [stencil_coefficients(2, dx) for dx in grid.spacing]
    clo = np.array([t[0] for t in taps])
    cmid = np.array([t[1] for t in taps])
    return clo, cmid, float(c**2)
