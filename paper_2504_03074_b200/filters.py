"""Filter configuration and the corrected filter constant — host-side mirror
of the hot-path part of waveholtz/filters.py.

Only what the explicit iteration consumes lives here: ``TimeMode`` and
``FilterConfig`` (filters.py:49-116), ``alpha_d`` (filters.py:160-166) and the
exception types the drivers raise (filters.py:55-60).  The closed-form filter
theory (beta, beta_d, predict_rate, filters.py:119-288) is out of scope
 — it is not executed per grid point.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

__all__ = ["TimeMode", "FilterConfig", "ResonanceError", "ExplicitStabilityError", "alpha_d", "mode_name"]


class TimeMode(Enum):
    CONTINUOUS = "continuous"
    EXPLICIT = "explicit"
    IMPLICIT = "implicit"


class ResonanceError(ValueError):
    """An eigenvalue coincides with the target frequency (filters.py:55-56)."""


class ExplicitStabilityError(ValueError):
    """lambda*dt exceeds the explicit stability limit (filters.py:59-60)."""


def mode_name(mode) -> str:
    """'explicit' / 'implicit' / 'continuous' from this package's or the reference's TimeMode."""
    return str(getattr(mode, "value", mode)).lower()


def _as_mode(mode) -> TimeMode:
    return mode if isinstance(mode, TimeMode) else TimeMode(mode_name(mode))


@dataclass(frozen=True)
class FilterConfig:
    """omega, periods N_p, steps per period N_t, time mode, optional alpha (filters.py:67-116)."""

    omega: float
    periods: int = 1
    steps_per_period: int = 10
    mode: TimeMode = TimeMode.IMPLICIT
    alpha: float | None = None

    def __post_init__(self):
        object.__setattr__(self, "mode", _as_mode(self.mode))
        if not self.omega > 0:
            raise ValueError("omega must be positive")
        if self.periods < 1 or self.steps_per_period < 1:
            raise ValueError("periods and steps_per_period must be positive")
        if self.mode is TimeMode.IMPLICIT and self.steps_per_period < 5:
            raise ValueError("implicit filtering needs at least 5 time-steps per period")

    @property
    def period(self) -> float:
        return 2.0 * math.pi / self.omega

    @property
    def total_time(self) -> float:
        return self.periods * self.period

    @property
    def dt(self) -> float:
        return self.period / self.steps_per_period

    @property
    def total_steps(self) -> int:
        return self.periods * self.steps_per_period

    @property
    def resolved_alpha(self) -> float:
        if self.alpha is not None:
            return self.alpha
        if self.mode is TimeMode.CONTINUOUS:
            return 0.5
        return alpha_d(2.0 * math.pi / self.steps_per_period)


def alpha_d(omega_dt: float) -> float:
    """tan(x/2)/tan(x) at x = omega*dt, x in (0, pi/2) (filters.py:160-166)."""
    if not 0.0 < omega_dt < math.pi / 2.0:
        raise ValueError(f"omega*dt = {omega_dt:.6g} outside (0, pi/2); need at least 5 steps per period")
    return math.tan(omega_dt / 2.0) / math.tan(omega_dt)
