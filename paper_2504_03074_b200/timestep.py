"""Explicit leapfrog stepping and the filtered wave solve on the GPU —
drop-in for the explicit branch of waveholtz/timestep.py.

Host side (this module): the time correction (timestep.py:41-97) and the
per-step scalar schedule, formed with the reference's own Python expressions
 so the device never evaluates a transcendental.
Device side (libwhb200.so): the fused leapfrog + filter kernel.

The implicit trapezoidal scheme (timestep.py:100-108, 148-247) runs on the
device too (``implicit.py``: CG with a multigrid / tridiagonal
preconditioner).  There is no CPU fallback.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .device import device_problem
from .filters import ExplicitStabilityError, TimeMode, alpha_d, mode_name
from .grid import GridField
from .implicit import correct_implicit, implicit_solver_for, implicit_wave_solve

__all__ = [
    "TimeCorrection", "WaveState", "correct_explicit", "correct_implicit", "cfl_constant", "step_explicit",
    "wave_solve_filtered", "time_schedule",
]

#: Courant numbers of leap-frog with order-p space discretisation (timestep.py:41-43).
#: Module-level and mutable like the reference's, so BASELINE's "CFL 0.9" is
#: ``_COURANT[2] = 0.9`` in both packages.
_COURANT = {2: 1.0, 4: math.sqrt(3.0) / 2.0}


def cfl_constant(p: int) -> float:
    return _COURANT[p]


@dataclass(frozen=True)
class TimeCorrection:
    """Corrected driving frequency and step (timestep.py:50-75)."""

    mode: TimeMode
    omega: float
    omega_tilde: float
    dt: float
    steps_per_period: int

    def __post_init__(self):
        nt, dt = self.steps_per_period, self.dt
        if abs(nt * dt - self.period_tilde) > 1e-13 * self.period_tilde:
            raise AssertionError("N_t*dt must equal the corrected period")
        if mode_name(self.mode) == "explicit":
            lhs = math.sin(self.omega_tilde * dt / 2.0) / (dt / 2.0)
            if abs(lhs - self.omega) > 1e-13 * self.omega:
                raise AssertionError("sin(w_e dt/2)/(dt/2) must equal omega")
        elif mode_name(self.mode) == "implicit":
            if nt < 5:
                raise AssertionError("implicit stepping needs N_t >= 5")
            if abs(math.cos(self.omega_tilde * dt) * (1.0 + (self.omega * dt) ** 2 / 2.0) - 1.0) > 1e-13:
                raise AssertionError("cos(w_i dt)(1 + (w dt)^2/2) must equal 1")

    @property
    def period_tilde(self) -> float:
        return 2.0 * math.pi / self.omega_tilde

    @property
    def alpha(self) -> float:
        return alpha_d(self.omega_tilde * self.dt)


def correct_explicit(omega: float, grid, p: int, c: float) -> TimeCorrection:
    """Smallest N_t >= 5 with c^2 dt^2 sum(1/dx^2) < C_p^2, dt = (2/w) sin(pi/N_t),
    w_e = 2 pi/(N_t dt) (timestep.py:78-97)."""
    if not omega > 0:
        raise ValueError("omega must be positive")
    inv_sq = sum(1.0 / dx**2 for dx in grid.spacing)
    bound = cfl_constant(p) ** 2
    n_t = max(5, math.ceil(2.0 * math.pi / omega / math.sqrt(bound / (c**2 * inv_sq))))
    dt = (2.0 / omega) * math.sin(math.pi / n_t)
    while not c**2 * dt**2 * inv_sq < bound:
        n_t += 1
        dt = (2.0 / omega) * math.sin(math.pi / n_t)
    return TimeCorrection(TimeMode.EXPLICIT, omega, 2.0 * math.pi / (n_t * dt), dt, n_t)


def time_schedule(corr, config) -> dict:
    """Per-step scalars of one filtered solve, formed exactly as the reference forms them.

    n_total = N_p*N_t (timestep.py:273); step n>0 forcing factor cos(wt*t^n) with
    t^n = n*dt (timestep.py:139, 144); filter weights (cos(wt*t^n) - alpha/2)*sigma_n
    with sigma = 1/2 at both ends (timestep.py:284, 297-298); first step uses
    0.5*dt**2, later steps dt**2 (timestep.py:137, 140); output scale (2/t_bar)*dt
    with t_bar = n_total*dt (timestep.py:277, 300).
    """
    n_total = config.periods * corr.steps_per_period
    dt = corr.dt
    wt = corr.omega_tilde
    alpha = corr.alpha
    cos_f = np.empty(n_total)
    cos_f[0] = 1.0  # the first step carries no cos factor
    acc_c = np.empty(n_total + 1)
    acc_c[0] = (math.cos(0.0) - 0.5 * alpha) * 0.5
    for n in range(1, n_total + 1):
        t = n * dt
        cs = math.cos(wt * t)
        if n < n_total:
            cos_f[n] = cs
        acc_c[n] = (cs - 0.5 * alpha) * (0.5 if n == n_total else 1.0)
    return {
        "n_total": n_total,
        "half_dt2": 0.5 * dt**2,
        "dt2": dt**2,
        "cos_f": cos_f,
        "acc_c": acc_c,
        "out_scale": (2.0 / (n_total * dt)) * dt,
    }


def _check_modes(config, corr):
    """timestep.py:266-269."""
    if mode_name(corr.mode) != mode_name(config.mode):
        raise ValueError(f"correction mode {corr.mode} does not match config mode {config.mode}")
    if mode_name(config.mode) == "implicit" and corr.steps_per_period != config.steps_per_period:
        raise ValueError("correction and config disagree on steps per period")
    if mode_name(config.mode) not in ("explicit", "implicit"):
        raise ValueError("the continuous filter cannot be time-stepped; pick explicit or implicit")


def _field_type(v):
    return type(v) if hasattr(type(v), "from_values") else GridField


def new_field(ftype, grid, ghost):
    """(field, writable interior view) of a freshly allocated field of type ``ftype`` (ours or the
    reference's GridField) backed by a recycled page-locked buffer, or None when the type does not
    expose its buffer."""
    try:
        fld = ftype(grid, ghost=ghost)
        _pin_storage(fld)
        return fld, fld._writable()
    except (AttributeError, TypeError):
        return None


def field_from_device(ftype, grid, ghost, ctx, field_id):
    """A freshly allocated field of type ``ftype`` (ours or the reference's GridField) holding
    device field ``field_id``: copied straight into the new field's (possibly ghost-padded)
    buffer with one strided D2H copy, no host-side repacking.  The device field's Dirichlet
    points are 0 by invariant, so the field is in the state set_values would leave it in."""
    made = new_field(ftype, grid, ghost)
    if made is None:
        return ftype.from_values(grid, ctx.download(field_id), ghost=ghost)
    fld, buf = made
    ctx.download_into(field_id, buf)
    fld._touch()
    return fld


def _pin_storage(fld):
    """Back a freshly made field by a recycled page-locked buffer (_native.PinnedPool), so its D2H
    copy -- and its H2D copy when it is the next call's input -- run at full PCIe rate.  Our
    GridField keeps its values unpadded (``_vals``); the reference's keeps a ghost-padded ``_buf``
    (grid.py:197-206), whose ghost frame is zeroed here as its constructor would have left it.
    Fields of other layouts keep their own storage."""
    pool = _native.pinned_pool()
    try:
        if isinstance(getattr(fld, "_vals", None), np.ndarray) and not hasattr(fld, "_buf"):
            fld._vals = pool.empty(fld._vals.shape)
            return
        if not isinstance(getattr(fld, "_buf", None), np.ndarray):
            return
        old = fld._buf
        new = pool.empty(old.shape)
    except (RuntimeError, MemoryError):  # no page-locked memory / pool full: keep pageable storage
        return
    g = int(getattr(fld, "ghost", 0))
    if g > 0:  # ghost frame := 0 (the interior is overwritten by the download)
        for ax in range(new.ndim):
            lo = [slice(None)] * new.ndim
            lo[ax] = slice(0, g)
            new[tuple(lo)] = 0.0
            lo[ax] = slice(new.shape[ax] - g, None)
            new[tuple(lo)] = 0.0
    fld._buf = new


def wave_solve_filtered(v, f, config, corr, op, linear_solver=None, implicit_first_step=True):
    """One application of W(v, f) on the GPU (timestep.py:250-301, explicit branch).

    Inputs are never mutated; a freshly allocated field of the input's type is
    returned with its Dirichlet boundary zeroed (timestep.py:301).  Implicit mode
    marches the trapezoidal scheme with the device CG solver (implicit.py); a
    ``linear_solver`` passed in (e.g. the reference's _ImplicitSolver, which its
    drivers hand over) is not used for arithmetic, but its ``inner`` counter is
    advanced by the device solver's iterations so run records stay meaningful."""
    _check_modes(config, corr)
    grid = op.grid
    dp = device_problem(grid, c=op.c, order=op.order)
    if mode_name(config.mode) == "implicit":
        own = getattr(linear_solver, "device_solver", None)
        solver = own if own is not None else implicit_solver_for(dp, grid, op.order, op.c, corr.dt)
        dp.set_forcing_field(f)
        dp.ctx.upload_view(_native.V, v.values)
        its = implicit_wave_solve(dp, solver, corr, time_schedule(corr, config), _native.V, _native.F,
                                  _native.OUT, implicit_first_step=implicit_first_step)
        if linear_solver is not None and hasattr(linear_solver, "inner"):
            linear_solver.inner += its
        return field_from_device(_field_type(v), grid, max(2, op.ghost_width), dp.ctx, _native.OUT)
    dp.set_schedule(time_schedule(corr, config))
    zero_f = dp.set_forcing_field(f)
    ctx = dp.ctx
    vals = v.values
    made = new_field(_field_type(v), grid, max(2, op.ghost_width))
    if made is not None and ctx.nbatch == 1 and ctx._strides(vals) is not None and ctx._strides(made[1]) is not None:
        # host field in, host field out in one call (whb_solve_host): on the three-step plan the
        # transfers of v and W(v, f) move in bands of rows behind the passes
        fld, buf = made
        ctx.solve_host(vals, buf, _native.OUT_PLAIN, zero_forcing=zero_f)
        fld._touch()
        return fld
    ctx.upload_view(_native.V, vals)
    ctx.filtered_solve(_native.OUT_PLAIN, zero_forcing=zero_f)
    return field_from_device(_field_type(v), grid, max(2, op.ghost_width), ctx, _native.OUT)


@dataclass
class WaveState:
    """Marching state of one solve (timestep.py:111-129)."""

    w: np.ndarray
    w_prev: np.ndarray
    n: int = 0
    t: float = 0.0
    accumulator: np.ndarray | None = None
    inner_iterations: int = 0

    @classmethod
    def start(cls, v: np.ndarray) -> "WaveState":
        w = np.array(v, dtype=float)
        return cls(w=w, w_prev=np.zeros_like(w))


def step_explicit(state: WaveState, op, f: np.ndarray, corr) -> WaveState:
    """One leapfrog step of host arrays on the GPU (timestep.py:132-145).

    Uses the step-level device API: W^n goes in the level buffer the kernel
    reads at step s (s = 0 for the start step, s = 2 otherwise; level L >= 1
    lives in slot L mod 4: WA, WB, WC, WD) with a
    one-off schedule whose cos factor is cos(wt*t^n)."""
    dt = corr.dt
    dp = device_problem(op.grid, c=op.c, order=op.order)
    ctx = dp.ctx
    cos_n = math.cos(corr.omega_tilde * state.t)
    sched = {"n_total": 4, "half_dt2": 0.5 * dt**2, "dt2": dt**2,
             "cos_f": np.array([1.0, 1.0, cos_n, 1.0]), "acc_c": np.zeros(5), "out_scale": 1.0}
    dp.set_schedule(sched)
    zero_f = dp.set_forcing(f)
    if state.n == 0:
        ctx.upload(_native.V, state.w)
        s, out_field = 0, _native.WA
    else:
        ctx.upload(_native.WB, state.w)       # level 2
        ctx.upload(_native.WA, state.w_prev)  # level 1
        s, out_field = 2, _native.WC          # level 3
    ctx.solve_begin(_native.OUT_PLAIN, zero_forcing=zero_f)
    ctx.step(s, 0)
    ctx.solve_end()
    w_next = ctx.download(out_field)
    state.w_prev = state.w
    state.w = w_next
    state.n += 1
    state.t = state.n * dt
    return state


def explicit_stability_check(lam_max: float, dt: float):
    """lambda*dt <= 2 (filters.py:205-215)."""
    if lam_max * dt / 2.0 > 1.0:
        raise ExplicitStabilityError(f"lambda*dt = {lam_max * dt:.6g} > 2")


def step_implicit(state: WaveState, op, f: np.ndarray, corr, linear_solver) -> WaveState:
    """One trapezoidal step (timestep.py:148-170): (I - (dt^2/2) L) W^{n+1} = rhs, the first
    step included (W^{-1} eliminated).  The reference's host expressions for rhs / guess, the
    Laplacian of W^{n-1} on the device (DiscreteOperator.apply_values), and the solve by
    ``linear_solver`` (make_implicit_solver: on the device)."""
    dt = corr.dt
    cos_fac = math.cos(corr.omega_tilde * dt)
    if state.n == 0:
        rhs = state.w - 0.5 * dt**2 * cos_fac * f
        guess = state.w
    else:
        lap_prev = op.apply_values(state.w_prev)
        force = f * (math.cos(corr.omega_tilde * state.t) * cos_fac)
        rhs = 2.0 * state.w - state.w_prev + 0.5 * dt**2 * lap_prev - dt**2 * force
        guess = 2.0 * state.w - state.w_prev
    w_next, iters = linear_solver(rhs, guess)
    state.inner_iterations = getattr(state, "inner_iterations", 0) + iters
    state.w_prev = state.w
    state.w = w_next
    state.n += 1
    state.t = state.n * dt
    return state
