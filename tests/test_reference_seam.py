"""CPU: the drop-in seam of INTEGRATION.md §1 — rebinding the reference's
``waveholtz.driver.wave_solve_filtered`` (imported by name at driver.py:38) to
this package's function reroutes the reference's own ``fpi_solve`` /
``krylov_solve``, with reference GridField / FilterConfig / TimeCorrection /
DiscreteOperator objects going in and reference GridFields coming out.

Runs in the build container (the reference is importable here, not on the
GPU box).  The device layer is replaced by a test double that computes with
the oracle, so what is checked is the host-side contract: argument handling,
scalar schedule, return type, and that the reference's own drivers produce
the same run as without the rebinding."""

import numpy as np
import pytest

import paper_2504_03074_b200 as wh
from paper_2504_03074_b200 import _native
from paper_2504_03074_b200 import timestep as ts
from oracle import reference_harness as RH
from oracle import waveholtz_oracle as O

pytestmark = pytest.mark.skipif(not RH.available(), reason="reference not present")


class FakeCtx:
    """Test double of _native.Context (oracle arithmetic, host memory)."""

    nbatch = 1

    def __init__(self, grid):
        self.grid = grid
        self.fields = {}
        self.sched = None
        self.host_solves = 0

    def _strides(self, a):  # as _native.Context._strides: views with a contiguous last axis
        if not isinstance(a, np.ndarray) or a.dtype != np.float64 or a.ndim not in (2, 3) or a.strides[-1] != 8:
            return None
        return a.strides[0] // 8, a.strides[-2] // 8

    def solve_host(self, v, out, out_mode=_native.OUT_PLAIN, zero_forcing=False):
        assert self._strides(v) is not None and self._strides(out) is not None and out.flags.writeable
        self.upload(_native.V, v)
        self.filtered_solve(out_mode, zero_forcing)
        out[...] = self.fields[_native.OUT]
        self.host_solves += 1
        return 0.0

    def set_schedule(self, member, sched):
        self.sched = sched

    def upload(self, field, values, member=0):
        self.fields[field] = np.array(values, dtype=float)

    def download(self, field, member=0, out=None):
        return np.array(self.fields[field])

    def upload_view(self, field, values, member=0):
        self.upload(field, values, member)

    def download_into(self, field, out, member=0):
        out[...] = self.fields[field]
        return out

    def filtered_solve(self, out_mode=_native.OUT_PLAIN, zero_forcing=False):
        f = np.zeros_like(self.fields[_native.V]) if zero_forcing else self.fields[_native.F]
        bcs = [getattr(b, "value", b) for b in self.grid.bcs]
        out = O.wave_solve_filtered(self.fields[_native.V], f, self.grid.spacing, self.sched, 1.0, bcs, 2)
        self.fields[_native.OUT] = out if out_mode == _native.OUT_PLAIN else self.fields[_native.V] - out
        return np.zeros(1)


class FakeProblem:
    def __init__(self, grid):
        self.ctx = FakeCtx(grid)
        self._sched = None

    def set_schedule(self, sched, member=0):
        self.ctx.set_schedule(member, sched)

    def set_forcing(self, values, member=0):
        self.ctx.upload(_native.F, values)
        return not np.any(values)

    def set_forcing_field(self, field, member=0):
        return self.set_forcing(field.values, member)


def test_rebinding_reroutes_the_reference_drivers(monkeypatch):
    ref = RH.import_reference()
    probs = {}
    monkeypatch.setattr(ts, "device_problem", lambda grid, c=1.0, order=2, device=0: probs.setdefault(
        id(grid), FakeProblem(grid)))
    with RH.courant(0.9):
        g = ref.grid.build_grid(2, ((0.0, 1.0), (0.0, 1.0)), (24, 20), "dirichlet")
        f = ref.driver.gaussian_source(g, 7.3, 50.0, 40.0, (0.4, 0.55))
        prob = ref.driver.HelmholtzProblem(g, 2, 1.0, 7.3, f)
        cfg = ref.filters.FilterConfig(omega=7.3, periods=1, steps_per_period=10, mode="explicit")
        v_ref, run_ref = ref.driver.fpi_solve(prob, cfg, tol=-1.0, maxit=6)
        x_ref, krun_ref = ref.driver.krylov_solve(prob, cfg, tol=1e-9)
        monkeypatch.setattr(ref.driver, "wave_solve_filtered", wh.wave_solve_filtered)
        v, run = ref.driver.fpi_solve(prob, cfg, tol=-1.0, maxit=6)
        x, krun = ref.driver.krylov_solve(prob, cfg, tol=1e-9)
    assert type(v) is ref.grid.GridField and type(x) is ref.grid.GridField
    assert np.array_equal(v.values, v_ref.values)
    assert run.residuals == run_ref.residuals
    assert krun.iterations == krun_ref.iterations
    assert np.array_equal(x.values, x_ref.values)
    assert probs, "the device layer was used"
    # 2D fields go in and out through the one-call host solve (strided reference buffers)
    assert all(p.ctx.host_solves > 0 for p in probs.values())


def test_reference_objects_accepted_directly(monkeypatch):
    ref = RH.import_reference()
    monkeypatch.setattr(ts, "device_problem", lambda grid, c=1.0, order=2, device=0: FakeProblem(grid))
    g = ref.grid.build_grid(1, (0.0, 1.0), 16, "dirichlet")
    op = ref.grid.DiscreteOperator(g, 2, 1.0)
    corr = ref.timestep.correct_explicit(5.5, g, 2, 1.0)
    cfg = ref.filters.FilterConfig(omega=5.5, periods=2, steps_per_period=corr.steps_per_period, mode="explicit")
    v = ref.grid.GridField.from_values(g, np.sin(np.linspace(0, 3, 17)))
    out = wh.wave_solve_filtered(v, ref.grid.GridField.zeros(g), cfg, corr, op)
    assert type(out) is ref.grid.GridField
    assert np.array_equal(out.values, ref.timestep.wave_solve_filtered(v, ref.grid.GridField.zeros(g), cfg, corr,
                                                                      op).values)
    bad = ref.filters.FilterConfig(omega=5.5, periods=1, steps_per_period=10, mode="implicit")
    with pytest.raises(ValueError, match="mode"):
        wh.wave_solve_filtered(v, v, bad, corr, op)
