"""Implicit (trapezoidal) WaveHoltz wave solves on the GPU — SURVEY §8(f) rank 4,
the implicit branch of waveholtz/timestep.py (148-247, 250-301) and the
solvers under it in waveholtz/linalg.py (62-99 CG, 189-346 multigrid,
380-421 tridiagonal).

Every step solves (I - (dt^2/2) c^2 L_h) W^{n+1} = rhs on device vectors of
the grid's whb context.  The solver is chosen exactly as the reference's
``_ImplicitSolver`` chooses it (timestep.py:183-212):

* 1D all-Dirichlet: the prefactored tridiagonal elimination — a direct solve
  for p = 2 (bitwise the reference's), the CG preconditioner for p = 4;
* 2D all-Dirichlet with cell counts that halve down to <= 8: CG
  preconditioned by one multigrid V-cycle (red-black Gauss-Seidel 2+2,
  full weighting, bilinear prolongation, dense coarse solve), captured as
  one CUDA graph;
* anything else (3D, periodic, uncoarsenable): plain CG.

The CG loop mirrors ``cg_solve``'s control flow on the host (convergence and
breakdown tests); each iteration's arithmetic — operator, V-cycle, dots and
the alpha/beta scalars — is one device graph (``whb_cg_iterate``) with one
readback of p.Ap and r.r.  Elementwise
values follow the reference's operation order; dots use the device's
fixed-order tree instead of BLAS, so iterates agree with the reference to the
inner tolerance (1e-12 relative per solve), not bitwise — the contract is
<= 1e-10 relative max-norm per WaveHoltz iterate (BASELINE north_star).
"""

from __future__ import annotations

import math

import numpy as np

from . import _native
from .filters import TimeMode

__all__ = ["correct_implicit", "DeviceImplicitSolver", "implicit_solver_for", "implicit_wave_solve"]


def correct_implicit(omega: float, n_t: int):
    """dt = (1/omega) sqrt(2/cos(2 pi/N_t) - 2), omega_i = 2 pi/(N_t dt) (timestep.py:100-108)."""
    from .timestep import TimeCorrection

    if n_t <= 4:
        raise ValueError("implicit time-stepping needs at least 5 time-steps per period")
    if not omega > 0:
        raise ValueError("omega must be positive")
    dt = math.sqrt(2.0 / math.cos(2.0 * math.pi / n_t) - 2.0) / omega
    omega_i = 2.0 * math.pi / (n_t * dt)
    return TimeCorrection(TimeMode.IMPLICIT, omega, omega_i, dt, n_t)


def _all_dirichlet(grid) -> bool:
    return all(str(getattr(b, "value", b)) == "dirichlet" for b in grid.bcs)


def _tridiag_factors(n_cells: int, dx: float, dt: float, c: float):
    """_ImplicitSolver._tridiag + TridiagFactorization.__init__ (timestep.py:214-221,
    linalg.py:380-407), same float operations: returns (sub, dp, cp)."""
    g = 0.5 * dt**2 * c**2 / dx**2
    n = n_cells - 1
    diag = np.full(n, 1.0 + 2.0 * g)
    off = np.full(n - 1, -g)
    cp = np.empty(n - 1)
    dp = np.empty(n)
    dp[0] = diag[0]
    if dp[0] == 0.0:
        raise ZeroDivisionError("zero pivot in tridiagonal factorization")
    for i in range(1, n):
        cp[i - 1] = off[i - 1] / dp[i - 1]
        piv = diag[i] - off[i - 1] * cp[i - 1]
        if piv == 0.0:
            raise ZeroDivisionError(f"zero pivot at row {i}")
        dp[i] = piv
    return off, dp, cp


def _second_difference(n_cells: int, dx: float) -> np.ndarray:
    m = n_cells - 1
    t = np.zeros((m, m))
    s = np.array([1.0, -2.0, 1.0]) / dx**2  # stencil_coefficients(2, dx) (grid.py:302-306)
    for i in range(m):
        t[i, i] = s[1]
        if i > 0:
            t[i, i - 1] = s[0]
        if i < m - 1:
            t[i, i + 1] = s[2]
    return t


def multigrid_levels(grid, c: float, dt: float):
    """MultigridHierarchy.__init__ (linalg.py:289-319): per level (cells, gamma, diag) and the
    inverse of the coarsest interior matrix I - (dt^2/2) c^2 L_2h.  Raises ValueError when
    the cells cannot halve down to <= 8 per axis (the reference then uses plain CG)."""
    coef = 0.5 * dt**2 * c**2
    cells = list(grid.cells)
    spacing = list(grid.spacing)
    levels = []
    while True:
        gamma = tuple(coef / dx**2 for dx in spacing)
        levels.append((tuple(cells), gamma, 1.0 + 2.0 * sum(gamma)))
        if any(n <= 8 for n in cells):
            break
        if any(n % 2 for n in cells):
            raise ValueError(f"grid cells {tuple(cells)} cannot be coarsened evenly to <= 8 per axis")
        cells = [n // 2 for n in cells]
        spacing = [2.0 * dx for dx in spacing]
    tx, ty = _second_difference(cells[0], spacing[0]), _second_difference(cells[1], spacing[1])
    lap = c**2 * (np.kron(tx, np.eye(ty.shape[0])) + np.kron(np.eye(tx.shape[0]), ty))
    a_coarse = np.eye(lap.shape[0]) - 0.5 * dt**2 * lap
    return levels, np.linalg.inv(a_coarse)


class DeviceImplicitSolver:
    """(I - (dt^2/2) c^2 L_h) w = rhs on device vectors (_ImplicitSolver, timestep.py:173-247)."""

    def __init__(self, ctx, grid, order: int, c: float, dt: float, tol: float = 1e-12, maxit: int = 400):
        self.ctx = ctx
        self.grid = grid
        self.order = order
        self.dt = dt
        self.tol = tol
        self.maxit = maxit
        self.inner = 0
        self.s = 0.5 * dt**2
        self.c = c
        self.tri = False
        self.precond = None
        self._tri_factors = None
        self._mg = None
        dirichlet = _all_dirichlet(grid)
        if grid.dim == 1 and dirichlet:
            self._tri_factors = _tridiag_factors(grid.cells[0], grid.spacing[0], dt, c)
            self.tri = True
        if grid.dim == 2 and dirichlet:
            try:
                levels, ainv = multigrid_levels(grid, c, dt)
            except ValueError:
                levels = None
            if levels is not None:
                # (a grid already <= 8 cells is a single-level hierarchy: its V-cycle is the dense solve)
                self._mg = ([lv[0] for lv in levels], [lv[1] for lv in levels], [lv[2] for lv in levels], ainv)
                self.precond = "mg"
        if grid.dim == 1 and self.tri and order == 4:
            self.precond = "tri"
        self.direct = self.tri and order == 2
        self.activate()
        (self.r, self.z, self.p, self.ap, self.tmp) = ctx.vec_reserve(5)

    def activate(self):
        """The context holds ONE tridiagonal factorisation / multigrid hierarchy (whb_tri_setup /
        whb_mg_setup replace it and drop the CG graphs that baked it): install this solver's
        (its dt) unless it is already the installed one.  Called before every solve, so solvers
        of different dt sharing a grid (omega A, B, A) never run on each other's factors."""
        if getattr(self.ctx, "_imp_active", None) is self:
            return
        if self._tri_factors is not None:
            self.ctx.tri_setup(*self._tri_factors)
        if self._mg is not None:
            self.ctx.mg_setup(*self._mg)
        self.ctx._imp_active = self

    def apply(self, x, y):
        """y = x - (0.5*dt**2) * c^2 L_h x  (timestep.py:225-226)."""
        self.ctx.imp_apply(x, y, self.s, self.tmp)

    def solve(self, rhs, guess, x) -> int:
        """x = A^{-1} rhs from the initial guess (cg_solve, linalg.py:62-99, or the direct
        tridiagonal solve); returns the iteration count and raises like the reference."""
        ctx = self.ctx
        self.activate()
        if self.direct:
            ctx.tri_solve(rhs, x)
            self.inner += 1
            return 1
        bnorm = math.sqrt(ctx.dot(rhs, rhs))
        if bnorm == 0.0:
            ctx.scale_into(0.0, rhs, x)
            return 0
        ctx.copy(guess, x)
        self.apply(x, self.ap)
        ctx.sub_into(rhs, self.ap, self.r)  # r = b - A(x)
        pre = {None: 0, "mg": 1, "tri": 2}[self.precond]
        z = self.r if pre == 0 else self.z
        # z = M r, p = z, rz = r.z on the device; rnorm = ||r||
        rnorm = math.sqrt(ctx.cg_begin(self.r, z, self.p, pre))
        k = 0
        converged = False
        for k in range(self.maxit):
            if rnorm <= self.tol * bnorm:
                converged = True
                break
            # Ap, alpha = rz/pAp, x += alpha p, r -= alpha Ap, z = M r, beta, p = z + beta p: one graph
            pap, rr = ctx.cg_iterate(x, self.r, z, self.p, self.ap, self.tmp, self.s, pre)
            if pap <= 0.0 or not math.isfinite(pap):
                break
            rnorm = math.sqrt(rr)
        else:
            k = self.maxit
            converged = rnorm <= self.tol * bnorm
        if not converged:
            raise RuntimeError(f"implicit solve did not reach {self.tol:g} "
                               f"(residual {rnorm / bnorm:.3e} after {k} iterations)")
        self.inner += k
        return k


def implicit_solver_for(dp, grid, order, c, dt, tol=1e-12, maxit=400) -> DeviceImplicitSolver:
    """One device solver (and its workspace) per (device problem, dt, tol), reused across solves."""
    cache = dp.__dict__.setdefault("_implicit", {})
    key = (float(dt), float(tol), int(maxit))
    if key not in cache:
        cache[key] = DeviceImplicitSolver(dp.ctx, grid, order, c, dt, tol=tol, maxit=maxit)
    solver = cache[key]
    solver.activate()
    return solver


class _Workspace:
    def __init__(self, ctx):
        ids = ctx.vec_reserve(8)
        self.w = ids[:3]           # time-level ring
        self.lap, self.rhs, self.guess, self.acc, self.zero = ids[3:]


def _workspace(dp) -> _Workspace:
    ws = dp.__dict__.get("_implicit_ws")
    if ws is None:
        ws = dp._implicit_ws = _Workspace(dp.ctx)
    return ws


def implicit_wave_solve(dp, solver: DeviceImplicitSolver, corr, sched: dict, v_id: int, f_id, out_id: int,
                        out_mode: int = _native.OUT_PLAIN, implicit_first_step: bool = True) -> int:
    """One implicit W(v, f) on device vectors (timestep.py:250-301, implicit branch).

    f_id None = zero forcing (waveholtz_operator).  out_mode OUT_PLAIN writes W(v, f) into
    out_id, OUT_AV writes v - W(v, 0) (driver.py:256-262).  Returns the inner iterations."""
    ctx = dp.ctx
    ws = _workspace(dp)
    if f_id is None:
        f_id = ws.zero  # a vector that is never written: exact zeros, like GridField.zeros
    dt = corr.dt
    wt = corr.omega_tilde
    n_total = sched["n_total"]
    acc_c = sched["acc_c"]
    cos_fac = math.cos(corr.omega_tilde * dt)
    prev, cur, nxt = ws.w
    ctx.copy(v_id, cur)                       # WaveState.start: w = copy(v), w_prev = 0
    ctx.copy(ws.zero, prev)
    ctx.scale_into(acc_c[0], cur, ws.acc)     # acc = ((cos 0 - alpha/2) * 0.5) * w
    inner0 = solver.inner
    for n in range(n_total):
        if n == 0 and not implicit_first_step:
            # explicit first step (timestep.py:288-292)
            ctx.apply_operator(cur, ws.lap)
            ctx.scale_into(math.cos(wt * dt), f_id, ws.guess)        # f * cos(wt*dt)
            ctx.sub_into(ws.lap, ws.guess, ws.rhs)                   # lap - f*cos
            ctx.copy(cur, nxt)
            ctx.axpy(0.5 * dt**2, ws.rhs, nxt)                        # w + (0.5*dt**2)*(...)
        else:
            # step_implicit (timestep.py:148-170); t = n*dt is the state's time before the step
            if n > 0:
                ctx.apply_operator(prev, ws.lap)
            fs = math.cos(corr.omega_tilde * (n * dt)) * cos_fac
            ctx.imp_rhs(cur, prev, ws.lap, f_id, ws.rhs, ws.guess, n == 0, 0.5 * dt**2 * cos_fac, 0.5 * dt**2,
                        dt**2, fs)
            solver.solve(ws.rhs, ws.guess, nxt)
        prev, cur, nxt = cur, nxt, prev
        ctx.axpy(acc_c[n + 1], cur, ws.acc)   # acc += ((cos(wt t) - alpha/2) sigma) * w
    ws.w = [prev, cur, nxt]
    if out_mode == _native.OUT_AV:
        ctx.scale_into(sched["out_scale"], ws.acc, ws.rhs)
        ctx.sub_into(v_id, ws.rhs, out_id)
    else:
        ctx.scale_into(sched["out_scale"], ws.acc, out_id)
    return solver.inner - inner0


class HostImplicitSolver:
    """make_implicit_solver's object (timestep.py:173-247, _ImplicitSolver): ``solver(rhs, guess)``
    solves (I - (dt^2/2) c^2 L_h) w = rhs for host arrays and returns (w, iterations); ``apply``
    is the operator; ``inner`` counts inner iterations.  The solve runs on the device (the same
    DeviceImplicitSolver the drivers use: tridiagonal elimination, MG- or tridiagonal-
    preconditioned CG), and wave_solve_filtered(linear_solver=this) uses ``device_solver``
    directly -- so the reference's driver, rebound onto this package, builds no
    CPU multigrid hierarchy."""

    def __init__(self, op, dt: float, tol: float = 1e-12, maxit: int = 400):
        from .device import device_problem

        self.op, self.dt, self.tol, self.maxit = op, float(dt), float(tol), int(maxit)
        self.inner = 0
        self._dp = device_problem(op.grid, c=op.c, order=op.order)
        self.device_solver = implicit_solver_for(self._dp, op.grid, op.order, op.c, self.dt, tol=self.tol,
                                                 maxit=self.maxit)
        self._ids = self._dp.ctx.vec_reserve(3)

    def apply(self, values: np.ndarray) -> np.ndarray:
        ctx = self._dp.ctx
        x, y, _ = self._ids
        ctx.vec_upload(x, np.asarray(values, dtype=float))
        self.device_solver.apply(x, y)
        return ctx.vec_download(y)

    def __call__(self, rhs: np.ndarray, guess: np.ndarray | None = None):
        ctx = self._dp.ctx
        r, g, x = self._ids
        ctx.vec_upload(r, np.asarray(rhs, dtype=float))
        ctx.vec_upload(g, np.zeros(np.shape(rhs)) if guess is None else np.asarray(guess, dtype=float))
        its = self.device_solver.solve(r, g, x)
        self.inner += its
        return ctx.vec_download(x), its


def make_implicit_solver(op, dt: float, tol: float = 1e-12) -> HostImplicitSolver:
    """timestep.py:246-247."""
    return HostImplicitSolver(op, dt, tol=tol)
