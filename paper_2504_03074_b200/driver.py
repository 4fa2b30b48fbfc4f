"""Fixed-point and GMRES WaveHoltz drivers on the GPU — drop-in for the
explicit-mode drivers of waveholtz/driver.py.

``fpi_solve`` keeps v, f and every wave-solve buffer resident on the device
for the whole iteration (the reference round-trips every iterate through new
numpy arrays, driver.py:221-227); the residual ||v_{k+1}-v_k||_2/sqrt(N) is
reduced inside the last leapfrog step of each pass.  ``krylov_solve`` runs
the reference's GMRES control flow over device vectors.  Deflation and the
direct sparse solve (driver.py:88-126, 303-343) are desk-scale oracles and
out of scope.
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, replace

import numpy as np

from . import _native
from .device import DeviceProblem, device_problem
from .filters import FilterConfig, ResonanceError, TimeMode, mode_name
from .grid import DiscreteOperator, GridField, bc_name
from .implicit import correct_implicit, implicit_solver_for, implicit_wave_solve
from .linalg import device_gmres
from .timestep import correct_explicit, field_from_device, time_schedule

__all__ = [
    "HelmholtzProblem", "WaveHoltzRun", "NearSingularError", "gaussian_source", "multi_gaussian_source",
    "fpi_solve", "krylov_solve", "waveholtz_operator", "apply_A", "measure_rate",
    "resolve_time_discretization", "resonance_gap", "HostFPIStep",
]


class NearSingularError(ValueError):
    """driver.py:58-59."""


def _axis_lambda2(n: int, dx: float, bc: str, order: int, c: float) -> np.ndarray:
    """lambda^2 of the 1D modes of one axis (grid.py:417-446): Dirichlet sines
    theta = m pi/n (m = 1..n-1), periodic Fourier theta = 2 pi m/n (m = 0..n/2);
    symbol 4 sin^2(theta/2) (+ its square / 12 at p = 4)."""
    m = np.arange(1, n) if bc == "dirichlet" else np.arange(0, n // 2 + 1)
    theta = m * np.pi / n if bc == "dirichlet" else 2.0 * np.pi * m / n
    s2 = 4.0 * np.sin(theta / 2.0) ** 2
    sym = s2 if order == 2 else s2 + s2**2 / 12.0
    return (c / dx) ** 2 * sym


def resonance_gap(grid, order: int, c: float, omega: float) -> float:
    """min |omega - lambda_h| / omega over the discrete spectrum (driver.py:72-81 with
    grid.py:417-472), without enumerating modes in Python: per-axis lambda^2 lists, the
    trailing axes combined into one sorted array, then a bisection per leading-axis value."""
    if order not in (2, 4):
        raise ValueError(f"unsupported order p={order}")
    per_axis = [_axis_lambda2(n, dx, bc_name(b), order, c) for n, dx, b in zip(grid.cells, grid.spacing, grid.bcs)]
    w2 = omega * omega
    if len(per_axis) == 1:
        lam = np.sqrt(per_axis[0])
        return float(np.min(np.abs(omega - lam)) / omega)
    tail = per_axis[-1]
    for arr in per_axis[-2:0:-1]:
        tail = np.add.outer(arr, tail).ravel()
    tail = np.sort(tail)
    best = np.inf
    for l0 in per_axis[0]:
        i = np.searchsorted(tail, w2 - l0)
        for j in (i - 1, i):
            if 0 <= j < tail.size:
                best = min(best, abs(omega - math.sqrt(l0 + tail[j])))
    return float(best / omega)


@dataclass(frozen=True)
class HelmholtzProblem:
    """L u + omega^2 u = f with homogeneous boundary data (driver.py:62-85)."""

    grid: object
    order: int
    c: float
    omega: float
    forcing: object

    def __post_init__(self):
        if not self.omega > 0:
            raise ValueError("omega must be positive")
        names = [bc_name(b) for b in self.grid.bcs]
        if all(b == "dirichlet" for b in names) or all(b == "periodic" for b in names):
            gap = resonance_gap(self.grid, self.order, self.c, self.omega)
            if gap < 1e-10:
                raise ResonanceError(f"omega = {self.omega:.12g} is within {gap:.1e} of a discrete eigenvalue")

    @property
    def operator(self) -> DiscreteOperator:
        return DiscreteOperator(self.grid, self.order, self.c)


@dataclass
class WaveHoltzRun:
    """Iteration diagnostics in the scaled 2h norm (driver.py:129-151)."""

    method: str
    periods: int
    residuals: list
    iterations: int
    converged: bool
    wall_time: float = 0.0
    inner_iterations: int = 0

    @property
    def wall_time_per_iteration(self) -> float:
        return self.wall_time / max(1, self.iterations)

    @property
    def cr(self) -> float:
        return measure_rate(self)[0]

    @property
    def ecr(self) -> float:
        return measure_rate(self)[1]


def measure_rate(run) -> tuple:
    """(CR, ECR) from the last five residual ratios (driver.py:154-160)."""
    r = [x for x in run.residuals if x > 0]
    if len(r) < 6:
        raise ValueError(f"need at least 6 positive residuals, have {len(r)}")
    cr = (r[-1] / r[-6]) ** 0.2
    return cr, cr ** (1.0 / run.periods)


def gaussian_source(grid, omega: float, a_g: float, b_g: float, x0) -> GridField:
    """a_g*exp(-b_g*|x-x0|^2) at the grid points (driver.py:163-179); r^2 is
    accumulated axis by axis from zeros, as the reference does, so the bits match."""
    x0 = np.atleast_1d(np.asarray(x0, dtype=float))
    if x0.size != grid.dim:
        raise ValueError(f"source center has {x0.size} coordinates for a {grid.dim}D grid")
    for (lo, hi), xc in zip(grid.bounds, x0):
        if not lo <= xc <= hi:
            raise ValueError(f"source center {xc} outside [{lo}, {hi}]")
    return GridField.from_values(grid, _gaussian_values(grid, a_g, b_g, x0))


def _gaussian_values(grid, a_g, b_g, x0, planes=None):
    """Values on planes [p0, p1) of axis 0 (all when None), memory-lean for 3D."""
    shape = tuple(grid.shape)
    p0, p1 = (0, shape[0]) if planes is None else planes
    sub = (p1 - p0,) + shape[1:]
    r2 = np.zeros(sub)
    for ax in range(grid.dim):
        lo = grid.bounds[ax][0]
        xs = lo + grid.spacing[ax] * np.arange(shape[ax])
        if ax == 0:
            xs = xs[p0:p1]
        bshape = [1] * grid.dim
        bshape[ax] = xs.size
        r2 = r2 + ((xs - x0[ax]) ** 2).reshape(bshape)
    return a_g * np.exp(-b_g * r2)


def multi_gaussian_source(grid, omega: float, n_gauss: int, seed: int = 0, slab_planes: int = 0) -> GridField:
    """BASELINE forcing recipe: rng = default_rng(seed);
    amp ~ U(-100,100,K), centres ~ U(0.1,0.9,(K,d)), widths ~ U(100,1000,K);
    f = sum_k gaussian_source(grid, omega, amp[k], b[k], centre[k]) in k order
    from zeros, boundary zeroed.  ``slab_planes`` > 0 evaluates the same
    per-element formula in axis-0 slabs to bound host memory on 1025^3."""
    rng = np.random.default_rng(seed)
    amp = rng.uniform(-100.0, 100.0, n_gauss)
    ctr = rng.uniform(0.1, 0.9, (n_gauss, grid.dim))
    wid = rng.uniform(100.0, 1000.0, n_gauss)
    shape = tuple(grid.shape)
    f = np.zeros(shape)
    step = slab_planes if slab_planes > 0 else shape[0]

    def slab(p0):
        p1 = min(shape[0], p0 + step)
        acc = np.zeros((p1 - p0,) + shape[1:])
        for k in range(n_gauss):
            g = _gaussian_values(grid, amp[k], wid[k], ctr[k], planes=(p0, p1))
            _zero_boundary_slab(grid, g, p0, p1)
            acc = acc + g
        f[p0:p1] = acc

    starts = range(0, shape[0], step)
    if len(starts) > 1:
        # slabs are independent and numpy's ufuncs release the GIL: host threads evaluate the same
        # per-element expressions (bitwise the same f), 1025^3 in seconds instead of minutes
        import concurrent.futures as cf

        workers = max(1, min(len(starts), os.cpu_count() or 1, 32))
        with cf.ThreadPoolExecutor(workers) as ex:
            list(ex.map(slab, starts))
    else:
        slab(0)
    return GridField.from_values(grid, f)


def _zero_boundary_slab(grid, a, p0, p1):
    for axis in range(grid.dim):
        sel = [slice(None)] * grid.dim
        if axis == 0:
            if p0 == 0:
                sel[0] = 0
                a[tuple(sel)] = 0.0
            if p1 == grid.shape[0]:
                sel[0] = -1
                a[tuple(sel)] = 0.0
        else:
            for edge in (0, -1):
                sel[axis] = edge
                a[tuple(sel)] = 0.0


def resolve_time_discretization(problem, config):
    """(corr, cfg): explicit mode derives N_t from stability (driver.py:182-192)."""
    if mode_name(config.mode) == "explicit":
        corr = correct_explicit(problem.omega, problem.grid, problem.order, problem.c)
        cfg = config
        if corr.steps_per_period != config.steps_per_period:
            cfg = replace(config, steps_per_period=corr.steps_per_period)
        return corr, cfg
    if mode_name(config.mode) == "implicit":
        return correct_implicit(problem.omega, config.steps_per_period), config
    raise ValueError("the continuous filter cannot be time-stepped; pick explicit or implicit")


def _device_for(problem) -> DeviceProblem:
    return device_problem(problem.grid, c=problem.c, order=problem.order)


def fpi_solve(problem, config, tol=1e-10, maxit=500, inner_tol=1e-12, device_state=None):
    """Fixed-point iteration from v = 0, stopping on the successive difference
    (driver.py:201-203, 211-244), device resident.

    tol < 0 runs exactly ``maxit`` passes with no host synchronisation between
    them; otherwise every pass is followed by the stopping test of
    driver.py:225-230 (sqrt(r)/sqrt(N) <= tol, the same IEEE operations) — on
    the host, or inside the kernel for cluster-resident grids."""
    corr, cfg = resolve_time_discretization(problem, config)
    dp = device_state or _device_for(problem)
    if mode_name(cfg.mode) == "implicit":
        return _fpi_implicit(problem, cfg, corr, dp, tol, maxit, inner_tol)
    dp.set_schedule(time_schedule(corr, cfg))
    dp.set_forcing_field(problem.forcing)
    dp.ctx.zero(_native.V)
    root_n = math.sqrt(problem.grid.size)
    residuals = []
    converged = False
    k = 0
    t0 = time.perf_counter()
    if tol < 0:
        rs = dp.ctx.fpi(maxit)
        residuals = [math.sqrt(x) / root_n for x in rs[:, 0]]
        k = len(residuals)
    else:
        rs = dp.ctx.fpi_scaled(maxit, tol, root_n)
        residuals = [math.sqrt(x) / root_n for x in rs[:, 0]]
        k = len(residuals)
        converged = k > 0 and residuals[-1] <= tol
    wall = time.perf_counter() - t0
    v = field_from_device(GridField, problem.grid, 2, dp.ctx, _native.V)
    run = WaveHoltzRun(method="fpi", periods=cfg.periods, residuals=residuals, iterations=k,
                       converged=converged, wall_time=wall, inner_iterations=0)
    return v, run


def _implicit_state(problem, dp, corr, inner_tol):
    solver = implicit_solver_for(dp, problem.grid, problem.order, problem.c, corr.dt, tol=inner_tol)
    ids = dp.__dict__.get("_implicit_fpi_ids")
    if ids is None:
        ids = dp._implicit_fpi_ids = dp.ctx.vec_reserve(2)
    return solver, ids


def _fpi_implicit(problem, cfg, corr, dp, tol, maxit, inner_tol):
    """_iterate (driver.py:211-244) with implicit wave solves, device resident: v, v_new and
    every solver vector stay on the GPU; the residual is a device reduction."""
    ctx = dp.ctx
    solver, (vnew, diff_id) = _implicit_state(problem, dp, corr, inner_tol)
    sched = time_schedule(corr, cfg)
    dp.set_forcing_field(problem.forcing)
    ctx.zero(_native.V)
    root_n = math.sqrt(problem.grid.size)
    residuals = []
    converged = False
    inner0 = solver.inner
    k = 0
    t0 = time.perf_counter()
    for k in range(1, maxit + 1):
        implicit_wave_solve(dp, solver, corr, sched, _native.V, _native.F, vnew)
        ctx.sub_into(vnew, _native.V, diff_id)
        diff = math.sqrt(ctx.dot(diff_id, diff_id)) / root_n   # np.linalg.norm(v_new - v)/sqrt(N)
        residuals.append(diff)
        ctx.copy(vnew, _native.V)
        if diff <= tol:
            converged = True
            break
    wall = time.perf_counter() - t0
    v = GridField.from_values(problem.grid, ctx.download(_native.V), ghost=2)
    run = WaveHoltzRun(method="fpi", periods=cfg.periods, residuals=residuals, iterations=k,
                       converged=converged, wall_time=wall, inner_iterations=solver.inner - inner0)
    return v, run


def waveholtz_operator(problem, config, corr=None, linear_solver=None, deflation=None):
    """Matrix-free A v = v - W(v, 0) on host arrays (driver.py:247-264); each call
    uploads v, runs one zero-forcing wave solve on the device and downloads A v."""
    if deflation is not None and len(deflation) > 0:
        raise NotImplementedError("deflation is out of scope for the GPU path (SURVEY §2)")
    if corr is None:
        corr, config = resolve_time_discretization(problem, config)
    dp = _device_for(problem)
    sched = time_schedule(corr, config)
    if mode_name(config.mode) == "implicit":
        solver, (xv, _) = _implicit_state(problem, dp, corr, 1e-12)

        def matvec_implicit(values: np.ndarray) -> np.ndarray:
            dp.ctx.vec_upload(xv, np.asarray(values, dtype=float))
            its = implicit_wave_solve(dp, solver, corr, sched, xv, None, _native.OUT, out_mode=_native.OUT_AV)
            if linear_solver is not None and hasattr(linear_solver, "inner"):
                linear_solver.inner += its
            return dp.ctx.download(_native.OUT)

        return matvec_implicit

    def matvec(values: np.ndarray) -> np.ndarray:
        dp.set_schedule(sched)
        dp.ctx.upload(_native.V, np.asarray(values, dtype=float))
        dp.ctx.filtered_solve(_native.OUT_AV, zero_forcing=True)
        return dp.ctx.download(_native.OUT)

    return matvec


def apply_A(v, problem, config, corr=None, linear_solver=None) -> GridField:
    """driver.py:267-270."""
    matvec = waveholtz_operator(problem, config, corr=corr, linear_solver=linear_solver)
    return GridField.from_values(problem.grid, matvec(np.array(v.values)))


def krylov_solve(problem, config, tol=1e-10, restart=50, maxit=500, deflation=None, inner_tol=1e-12):
    """GMRES on (I - S) v = b, b = W(0, f), residuals in the scaled norm
    (driver.py:273-300), every vector device resident."""
    if deflation is not None and len(deflation) > 0:
        raise NotImplementedError("deflation is out of scope for the GPU path (SURVEY §2)")
    corr, cfg = resolve_time_discretization(problem, config)
    dp = _device_for(problem)
    ctx = dp.ctx
    t0 = time.perf_counter()
    implicit = mode_name(cfg.mode) == "implicit"
    dp.set_forcing_field(problem.forcing)
    ctx.zero(_native.V)
    if implicit:
        solver, _ = _implicit_state(problem, dp, corr, inner_tol)
        inner0 = solver.inner
        sched = time_schedule(corr, cfg)
        implicit_wave_solve(dp, solver, corr, sched, _native.V, _native.F, _native.OUT)

        def mv(src, dst):
            implicit_wave_solve(dp, solver, corr, sched, src, None, dst, out_mode=_native.OUT_AV)
    else:
        dp.set_schedule(time_schedule(corr, cfg))
        ctx.filtered_solve(_native.OUT_PLAIN)  # OUT = b = W(0, f)   (driver.py:279-281)
        mv = ctx.matvec
    m = max(1, min(restart, maxit))
    ids = ctx.vec_reserve(m + 4) if not hasattr(dp, "_krylov_ids") or len(dp._krylov_ids) < m + 4 else dp._krylov_ids
    dp._krylov_ids = ids
    b_id, x_id, work = ids[0], ids[1], ids[2:]
    ctx.copy(_native.OUT, b_id)
    scale = math.sqrt(problem.grid.size)
    rep = device_gmres(ctx, mv, b_id, x_id, tol=0.0, atol=tol * scale, restart=restart, maxit=maxit,
                       work_ids=work)
    x = ctx.vec_download(x_id)
    wall = time.perf_counter() - t0
    run = WaveHoltzRun(method="gmres", periods=cfg.periods, residuals=[r / scale for r in rep.residual_history],
                       iterations=rep.iterations, converged=rep.converged, wall_time=wall,
                       inner_iterations=(solver.inner - inner0) if implicit else 0)
    return GridField.from_values(problem.grid, x), run


class HostFPIStep:
    """The body of the reference's fixed-point loop with host buffers
    (driver.py:222-226): ``diff = step(v_in, v_out)`` copies v_in to the device,
    runs one W(v, f) pass, copies v_new into v_out and returns
    ||v_new - v_in||_2 / sqrt(N).  Pass pinned arrays (``_native.PinnedBuffer``)
    for full-rate transfers; f stays resident after the first call."""

    def __init__(self, problem, config, inner_tol=1e-12, device_state=None):
        corr, cfg = resolve_time_discretization(problem, config)
        self.problem = problem
        self.config = cfg
        self.corr = corr
        self.dp = device_state or _device_for(problem)
        self.dp.set_schedule(time_schedule(corr, cfg))
        self.dp.set_forcing_field(problem.forcing)
        self._root_n = math.sqrt(problem.grid.size)
        self._implicit = None
        if mode_name(cfg.mode) == "implicit":
            self._implicit = _implicit_state(problem, self.dp, corr, inner_tol)
            self._sched = time_schedule(corr, cfg)

    def __call__(self, v_in: np.ndarray, v_out: np.ndarray) -> float:
        if v_in.shape != tuple(self.problem.grid.shape) or v_out.shape != v_in.shape:
            raise ValueError("v_in/v_out must have the grid shape")
        if not (v_in.flags.c_contiguous and v_out.flags.c_contiguous and v_out.flags.writeable):
            raise ValueError("v_in/v_out must be C-contiguous (v_out writeable)")
        if v_in.dtype != np.float64 or v_out.dtype != np.float64:
            raise ValueError("v_in/v_out must be float64 (the grid's dtype, grid.py:219)")
        if self._implicit is not None:
            ctx = self.dp.ctx
            solver, (vnew, diff_id) = self._implicit
            ctx.upload(_native.V, v_in)
            implicit_wave_solve(self.dp, solver, self.corr, self._sched, _native.V, _native.F, vnew)
            ctx.sub_into(vnew, _native.V, diff_id)
            d = math.sqrt(ctx.dot(diff_id, diff_id)) / self._root_n
            ctx.vec_download(vnew, out=v_out)
            return d
        return math.sqrt(self.dp.ctx.iterate_host(v_in, v_out)) / self._root_n
