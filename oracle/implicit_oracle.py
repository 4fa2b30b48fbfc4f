"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference's IMPLICIT
(trapezoidal) WaveHoltz path.

Only ``tests/`` and ``bench.py`` (the CPU baseline of the implicit workload)
may use this module, as the checker or the timed CPU baseline; the product
package never imports it.

Restates, in the reference's operation order:
  * correct_implicit                         timestep.py:100-108
  * step_implicit                            timestep.py:148-170
  * _ImplicitSolver (solver choice, apply)   timestep.py:173-247
  * cg_solve                                 linalg.py:62-99
  * multigrid V-cycle (RB Gauss-Seidel, full weighting, bilinear
    prolongation, dense coarse LU)           linalg.py:189-346
  * tridiagonal elimination                  linalg.py:380-421
  * the implicit branch of wave_solve_filtered  timestep.py:250-301
Pinned against golden outputs of the reference itself
(tests/golden/implicit.*, tests/test_oracle_implicit.py).  Third-party
arithmetic: numpy (BLAS dot/nrm2 in CG) and scipy.linalg.lu_factor/lu_solve
for the coarsest multigrid level, as in the reference.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.linalg

from .waveholtz_oracle import alpha_d, laplacian_general


def correct_implicit(omega: float, n_t: int):
    """timestep.py:100-108 -> (N_t, dt, omega_i)."""
    if n_t <= 4:
        raise ValueError("implicit time-stepping needs at least 5 time-steps per period")
    dt = math.sqrt(2.0 / math.cos(2.0 * math.pi / n_t) - 2.0) / omega
    return n_t, dt, 2.0 * math.pi / (n_t * dt)


def _cells(shape):
    return tuple(n - 1 for n in shape)


class Tridiag:
    """Prefactored Thomas elimination (linalg.py:380-421)."""

    def __init__(self, sub, diag, sup):
        n = diag.size
        self.n, self.sub = n, sub
        self.cp = np.empty(n - 1)
        self.dp = np.empty(n)
        self.dp[0] = diag[0]
        for i in range(1, n):
            self.cp[i - 1] = sup[i - 1] / self.dp[i - 1]
            self.dp[i] = diag[i] - sub[i - 1] * self.cp[i - 1]

    def solve(self, b):
        n = self.n
        y = np.empty(n)
        y[0] = b[0]
        for i in range(1, n):
            y[i] = b[i] - self.sub[i - 1] / self.dp[i - 1] * y[i - 1]
        x = np.empty(n)
        x[-1] = y[-1] / self.dp[-1]
        for i in range(n - 2, -1, -1):
            x[i] = y[i] / self.dp[i] - self.cp[i] * x[i + 1]
        return x


class Level:
    """One level of I - (dt^2/2) c^2 Lap_2h (linalg.py:198-275), 2D."""

    def __init__(self, cells, spacing, coef):
        self.cells = tuple(cells)
        self.gamma = tuple(coef / dx**2 for dx in spacing)
        self.diag = 1.0 + 2.0 * sum(self.gamma)
        self.shape = tuple(n + 1 for n in cells)

    def apply(self, u):
        gx, gy = self.gamma
        out = np.zeros_like(u)
        out[1:-1, 1:-1] = (self.diag * u[1:-1, 1:-1] - gx * (u[:-2, 1:-1] + u[2:, 1:-1])
                           - gy * (u[1:-1, :-2] + u[1:-1, 2:]))
        return out

    def colour(self, u, b, colour):
        gx, gy = self.gamma
        nx, ny = self.cells
        for pi in (0, 1):
            i0, j0 = 1 + pi, 1 + (colour + pi) % 2
            c = (slice(i0, nx, 2), slice(j0, ny, 2))
            n = (slice(i0 - 1, nx - 1, 2), slice(j0, ny, 2))
            s = (slice(i0 + 1, nx + 1, 2), slice(j0, ny, 2))
            w = (slice(i0, nx, 2), slice(j0 - 1, ny - 1, 2))
            e = (slice(i0, nx, 2), slice(j0 + 1, ny + 1, 2))
            u[c] = (b[c] + gx * (u[n] + u[s]) + gy * (u[w] + u[e])) / self.diag

    def restrict(self, r):
        mx, my = self.cells[0] // 2, self.cells[1] // 2
        rc = np.zeros((mx + 1, my + 1))
        ce = r[2:-1:2, 2:-1:2]
        edges = r[1:-2:2, 2:-1:2] + r[3::2, 2:-1:2] + r[2:-1:2, 1:-2:2] + r[2:-1:2, 3::2]
        corners = r[1:-2:2, 1:-2:2] + r[1:-2:2, 3::2] + r[3::2, 1:-2:2] + r[3::2, 3::2]
        rc[1:-1, 1:-1] = (4.0 * ce + 2.0 * edges + corners) / 16.0
        return rc

    def prolong(self, ec):
        e = np.zeros(self.shape)
        e[0::2, 0::2] = ec
        e[1::2, 0::2] = 0.5 * (ec[:-1, :] + ec[1:, :])
        e[0::2, 1::2] = 0.5 * (ec[:, :-1] + ec[:, 1:])
        e[1::2, 1::2] = 0.25 * (ec[:-1, :-1] + ec[1:, :-1] + ec[:-1, 1:] + ec[1:, 1:])
        return e


class Multigrid:
    """V-cycle preconditioner hierarchy (linalg.py:278-346), 2D all-Dirichlet."""

    def __init__(self, shape, spacing, c, dt, nu1=2, nu2=2):
        coef = 0.5 * dt**2 * c**2
        cells, sp = list(_cells(shape)), list(spacing)
        self.levels = []
        while True:
            self.levels.append(Level(cells, sp, coef))
            if any(n <= 8 for n in cells):
                break
            if any(n % 2 for n in cells):
                raise ValueError("cannot coarsen")
            cells = [n // 2 for n in cells]
            sp = [2.0 * d for d in sp]
        self.nu1, self.nu2 = nu1, nu2
        mats = []
        for n, d in zip(cells, sp):
            m = n - 1
            t = np.zeros((m, m))
            s = np.array([1.0, -2.0, 1.0]) / d**2
            for i in range(m):
                t[i, i] = s[1]
                if i:
                    t[i, i - 1] = s[0]
                if i < m - 1:
                    t[i, i + 1] = s[2]
            mats.append(t)
        lap = c**2 * (np.kron(mats[0], np.eye(mats[1].shape[0])) + np.kron(np.eye(mats[0].shape[0]), mats[1]))
        self._lu = scipy.linalg.lu_factor(np.eye(lap.shape[0]) - 0.5 * dt**2 * lap)
        self._coarse_shape = tuple(n + 1 for n in cells)

    def _coarse(self, b):
        out = np.zeros(self._coarse_shape)
        out[1:-1, 1:-1] = scipy.linalg.lu_solve(self._lu, np.ascontiguousarray(b[1:-1, 1:-1]).ravel()).reshape(
            out[1:-1, 1:-1].shape)
        return out

    def _cycle(self, lvl, b, u):
        L = self.levels[lvl]
        if lvl == len(self.levels) - 1:
            return self._coarse(b)
        for _ in range(self.nu1):
            L.colour(u, b, 0)
            L.colour(u, b, 1)
        r = b - L.apply(u)
        ec = self._cycle(lvl + 1, L.restrict(r), np.zeros(self.levels[lvl + 1].shape))
        u += L.prolong(ec)
        for _ in range(self.nu2):
            L.colour(u, b, 1)
            L.colour(u, b, 0)
        return u

    def __call__(self, r):
        return self._cycle(0, np.asarray(r, dtype=float), np.zeros(self.levels[0].shape))


def cg(apply, b, x0, tol, maxit, precond=None):
    """linalg.py:62-99 with x0 given; returns (x, iterations) or raises."""
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros_like(b), 0
    x = np.array(x0, dtype=float)
    r = b - apply(x)
    z = r if precond is None else precond(r)
    p = z.copy()
    rz = float(np.vdot(r, z))
    rnorm = np.linalg.norm(r)
    for k in range(maxit):
        if rnorm <= tol * bnorm:
            return x, k
        ap = apply(p)
        pap = float(np.vdot(p, ap))
        if pap <= 0.0 or not np.isfinite(pap):
            raise RuntimeError("CG breakdown")
        alpha = rz / pap
        x = x + alpha * p
        r = r - alpha * ap
        rnorm = np.linalg.norm(r)
        z = r if precond is None else precond(r)
        rz_new = float(np.vdot(r, z))
        p = z + (rz_new / rz) * p
        rz = rz_new
    if rnorm <= tol * bnorm:
        return x, maxit
    raise RuntimeError("CG did not converge")


class ImplicitSolver:
    """Solver choice of timestep.py:183-212 and its __call__ (timestep.py:228-247)."""

    def __init__(self, shape, spacing, bcs, order, c, dt, tol=1e-12, maxit=400):
        self.shape, self.spacing, self.bcs, self.order, self.c, self.dt = shape, spacing, bcs, order, c, dt
        self.tol, self.maxit, self.inner = tol, maxit, 0
        self.tri = self.precond = None
        dirichlet = all(b == "dirichlet" for b in bcs)
        if len(shape) == 1 and dirichlet:
            n = shape[0] - 1
            g = 0.5 * dt**2 * c**2 / spacing[0] ** 2
            off = np.full(n - 2, -g)
            self.tri = Tridiag(off, np.full(n - 1, 1.0 + 2.0 * g), off)
        if len(shape) == 2 and dirichlet:
            try:
                self.precond = Multigrid(shape, spacing, c, dt)
            except ValueError:
                self.precond = None
        if self.tri is not None and order == 4:
            tri = self.tri

            def tri_pre(r):
                out = np.zeros(shape)
                out[1:-1] = tri.solve(r[1:-1])
                return out

            self.precond = tri_pre

    def apply(self, u):
        return u - 0.5 * self.dt**2 * laplacian_general(u, self.spacing, self.bcs, self.order, self.c)

    def __call__(self, rhs, guess):
        if self.order == 2 and self.tri is not None:
            out = np.zeros(self.shape)
            out[1:-1] = self.tri.solve(rhs[1:-1])
            self.inner += 1
            return out
        x, its = cg(self.apply, rhs, guess, self.tol, self.maxit, self.precond)
        self.inner += its
        return x


def wave_solve_implicit(v, f, spacing, bcs, order, omega, n_t, c=1.0, solver=None, implicit_first_step=True,
                        max_steps=None):
    """The implicit branch of wave_solve_filtered (timestep.py:270-301), N_p = 1.
    ``max_steps`` stops after that many steps (a bounded timing sample; output then partial)."""
    n_t, dt, wt = correct_implicit(omega, n_t)
    alpha = alpha_d(wt * dt)
    solver = solver or ImplicitSolver(v.shape, spacing, bcs, order, c, dt)
    lap = lambda u: laplacian_general(u, spacing, bcs, order, c)  # noqa: E731
    w, w_prev = np.array(v, dtype=float), np.zeros_like(v)
    acc = (math.cos(0.0) - 0.5 * alpha) * 0.5 * w
    cos_fac = math.cos(wt * dt)
    t = 0.0
    for n in range(n_t if max_steps is None else min(n_t, max_steps)):
        if n == 0 and not implicit_first_step:
            w_next = w + 0.5 * dt**2 * (lap(w) - f * math.cos(wt * dt))
        elif n == 0:
            w_next = solver(w - 0.5 * dt**2 * cos_fac * f, w)
        else:
            rhs = 2.0 * w - w_prev + 0.5 * dt**2 * lap(w_prev) - dt**2 * (f * (math.cos(wt * t) * cos_fac))
            w_next = solver(rhs, 2.0 * w - w_prev)
        w_prev, w = w, w_next
        t = (n + 1) * dt
        sigma = 0.5 if n + 1 == n_t else 1.0
        acc += (math.cos(wt * t) - 0.5 * alpha) * sigma * w
    return (2.0 / (n_t * dt)) * dt * acc, solver
