"""Predicted WaveHoltz contraction rate (host math, small arrays): the reference's filter
theory that `waveholtz converge` prints next to the measured rate (summary.csv
``predicted_mu``).  Restated from filters.py:119-288 and grid.py:417-472 of the reference;
nothing here touches a grid-sized field.

    discrete_eigenvalues_symbolic(grid, p, c)   grid.py:417-472  sorted lambda_h of L_ph
    beta / sinc_d / beta_d                      filters.py:119-182
    lambda_tilde_explicit / _implicit           filters.py:205-222
    predict_rate                                filters.py:235-288
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .filters import ExplicitStabilityError, ResonanceError, TimeMode, _as_mode
from .grid import bc_name

__all__ = ["discrete_eigenvalues_symbolic", "beta", "sinc_d", "beta_d", "lambda_tilde_explicit",
           "lambda_tilde_implicit", "RatePrediction", "predict_rate"]

# symbol series coefficients B_mu of the order-p central difference (p = 2: [1]; p = 4: [1, 1/12])
_B_MU = (1.0, 1.0 / 12.0, 1.0 / 90.0, 1.0 / 560.0)


def _symbol(p: int, theta):
    s2 = 4.0 * np.sin(np.asarray(theta) / 2.0) ** 2
    acc = np.zeros_like(s2)
    for mu in range(p // 2):
        acc += _B_MU[mu] * s2 ** (mu + 1)
    return acc


def _axis_lambda2(grid, axis: int, p: int, c: float) -> list:
    n = grid.cells[axis]
    dx = grid.spacing[axis]
    if bc_name(grid.bcs[axis]) == "dirichlet":
        return [float((c / dx) ** 2 * _symbol(p, m * np.pi / n)) for m in range(1, n)]
    out = [0.0]
    for m in range(1, (n + 1) // 2):
        lam2 = float((c / dx) ** 2 * _symbol(p, 2.0 * np.pi * m / n))
        out += [lam2, lam2]
    if n % 2 == 0:
        out.append(float((c / dx) ** 2 * _symbol(p, np.pi)))
    return out


def discrete_eigenvalues_symbolic(grid, p: int, c: float = 1.0) -> np.ndarray:
    """Sorted eigenvalues lambda_h >= 0 with L_ph Phi = -lambda_h^2 Phi (all-Dirichlet or
    all-periodic grids; tensor sums of the per-axis symbols)."""
    kinds = {bc_name(b) for b in grid.bcs}
    if len(kinds) != 1:
        raise ValueError("mixed boundary conditions: use the dense eigensolver oracle")
    per_axis = [_axis_lambda2(grid, ax, p, c) for ax in range(grid.dim)]
    lam2 = np.array(per_axis[0])
    for more in per_axis[1:]:
        lam2 = np.add.outer(lam2, np.array(more)).ravel()
    return np.sort(np.sqrt(lam2), kind="stable")


def _sinc(x):
    return np.sinc(np.asarray(x) / np.pi)


def beta(lam, omega: float, t_bar: float, alpha: float = 0.5):
    """Continuous filter value (filters.py:123-131)."""
    lam = np.asarray(lam, dtype=float)
    val = _sinc((omega - lam) * t_bar) + _sinc((omega + lam) * t_bar) - alpha * _sinc(lam * t_bar)
    return float(val) if val.ndim == 0 else val


def sinc_d(z, T: float, dt: float):
    """Discrete sinc with its removable singularities taken as limits (filters.py:134-157)."""
    n_ratio = T / dt
    n = round(n_ratio)
    if n < 1 or abs(n_ratio - n) > 1e-9 * max(1.0, n):
        raise ValueError("sinc_d requires T to be an integer number of steps dt")
    phi = np.asarray(z, dtype=float) * dt / 2.0
    m = np.round(phi / np.pi)
    d = phi - m * np.pi
    tiny = np.abs(d) < 1e-300
    safe_d = np.where(tiny, 1.0, d)
    val = np.where(tiny, 1.0, np.sin(2.0 * n * safe_d) * np.cos(safe_d) / (2.0 * n * np.sin(safe_d)))
    return float(val) if np.ndim(val) == 0 else val


def beta_d(lam, omega: float, T: float, n_t: int, alpha: float):
    """Discrete (trapezoidal) filter value, three-sinc closed form (filters.py:169-182)."""
    dt = T / n_t
    lam = np.asarray(lam, dtype=float)
    val = sinc_d(omega + lam, T, dt) + sinc_d(omega - lam, T, dt) - alpha * sinc_d(lam, T, dt)
    return float(val) if np.ndim(val) == 0 else val


def lambda_tilde_explicit(lam_h, dt: float):
    """(2/dt) asin(lam dt/2) (filters.py:205-215)."""
    lam_h = np.asarray(lam_h, dtype=float)
    arg = lam_h * dt / 2.0
    if np.any(arg > 1.0):
        worst = float(np.max(lam_h))
        raise ExplicitStabilityError(f"lambda*dt = {worst * dt:.6g} > 2: mode {worst:.6g} is explicitly unstable")
    val = (2.0 / dt) * np.arcsin(arg)
    return float(val) if val.ndim == 0 else val


def lambda_tilde_implicit(lam_h, dt: float):
    """(1/dt) acos(1/(1 + (lam dt)^2/2)) (filters.py:218-222)."""
    lam_h = np.asarray(lam_h, dtype=float)
    val = (1.0 / dt) * np.arccos(1.0 / (1.0 + (lam_h * dt) ** 2 / 2.0))
    return float(val) if val.ndim == 0 else val


@dataclass(frozen=True)
class RatePrediction:
    mu: float
    argmax_index: int
    betas: np.ndarray
    non_contractive: tuple = ()


def predict_rate(lambdas_h, config, omega_tilde=None, alpha=None, deflated=()) -> RatePrediction:
    """mu = max |beta| over the mapped eigenvalues (filters.py:235-288)."""
    lambdas_h = np.asarray(lambdas_h, dtype=float)
    w = config.omega if omega_tilde is None else omega_tilde
    mode = _as_mode(config.mode)
    if mode is TimeMode.CONTINUOUS:
        mapped = lambdas_h
        a = 0.5 if (alpha is None and config.alpha is None) else (config.resolved_alpha if alpha is None else alpha)
        t_bar = config.periods * 2.0 * math.pi / w
        betas = np.atleast_1d(beta(mapped, w, t_bar, a))
    else:
        dt = 2.0 * math.pi / (w * config.steps_per_period)
        if mode is TimeMode.EXPLICIT:
            mapped = np.atleast_1d(lambda_tilde_explicit(lambdas_h, dt))
        else:
            mapped = np.atleast_1d(lambda_tilde_implicit(lambdas_h, dt))
        a = config.resolved_alpha if alpha is None else alpha
        t_bar = config.periods * 2.0 * math.pi / w
        betas = np.atleast_1d(beta_d(mapped, w, t_bar, config.total_steps, a))
    close = np.abs(mapped - w) <= 1e-12 * abs(w)
    if np.any(close):
        bad = int(np.argmax(close))
        raise ResonanceError(f"eigenvalue {lambdas_h.flat[bad]:.15g} maps onto the driving frequency {w:.15g}")
    deflated = set(int(i) for i in deflated)
    mu, argmax = -1.0, -1
    for i, b in enumerate(np.abs(betas)):
        if i in deflated:
            continue
        if b > mu:
            mu, argmax = float(b), i
    if argmax < 0:
        raise ValueError("no eigenvalues left after deflation")
    non_contractive = tuple(int(i) for i in np.nonzero(np.abs(betas) >= 1.0)[0] if i not in deflated)
    return RatePrediction(mu=mu, argmax_index=argmax, betas=betas, non_contractive=non_contractive)
