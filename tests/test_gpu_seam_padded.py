"""GPU: the Python seam with fields in the REFERENCE's storage layout.

The reference's GridField keeps its values inside a ghost-padded buffer (grid.py:185-227: ``_buf``
of shape n + 2 * ghost per axis, ``values`` a read-only view of the interior), so what
``wave_solve_filtered`` hands to the C ABI are strided views on both sides.  The reference is not
importable on the GPU box; ``PaddedField`` below is a stand-in with the same storage contract
(constructor, ``_buf``, ``values``, ``_writable``, ``_touch``, ``from_values``).  Checked: 2D
(serial host solve, strided 3D copies) and 3D on the three-step plan with the banded host solve
forced (strided band copies), two chained calls each, interior bitwise equal to the C restatement,
result of the input's type with a zero ghost frame."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import json, sys, numpy as np
sys.path.insert(0, %(root)r)
import paper_2504_03074_b200 as wh
from paper_2504_03074_b200 import timestep as ts
from oracle import native as ON, waveholtz_oracle as O
ts._COURANT[2] = 0.9


class PaddedField:
    def __init__(self, grid, ghost=2, values=None):
        self.grid, self.ghost = grid, int(ghost)
        self._buf = np.zeros(tuple(n + 2 * self.ghost for n in grid.shape))
        self.generation = 0
        if values is not None:
            self._writable()[...] = values
            self.generation += 1

    def _core(self):
        return tuple(slice(self.ghost, self.ghost + n) for n in self.grid.shape)

    @property
    def values(self):
        v = self._buf[self._core()]
        v.flags.writeable = False
        return v

    def _writable(self):
        v = self._buf[self._core()]
        v.flags.writeable = True
        return v

    def _touch(self):
        self.generation += 1

    @classmethod
    def from_values(cls, grid, values, ghost=2):
        return cls(grid, ghost, values)


out = []
for cells, omega in %(cases)r:
    d = len(cells)
    g = wh.build_grid(d, [(0.0, 1.0)] * d, list(cells), "dirichlet")
    f = wh.multi_gaussian_source(g, omega, 3, seed=6)
    corr = wh.correct_explicit(omega, g, 2, 1.0)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    op = wh.DiscreteOperator(g, 2, 1.0)
    v0 = np.array(wh.GridField.from_values(g, np.random.default_rng(8).standard_normal(g.shape) * 1e-3).values)
    v = PaddedField(g, 3, v0)
    fp = PaddedField(g, 2, np.array(f.values))
    ref, mis, frame, types = v0, 0, 0.0, []
    ctx = wh.device.device_problem(g).ctx
    launches = []
    for it in range(2):
        l0 = ctx.launch_count()
        w = wh.wave_solve_filtered(v, fp, cfg, corr, op)
        launches.append(ctx.launch_count() - l0)
        ref = ON.wave_solve(ref, np.array(f.values), g.spacing, sc)
        mis += int(np.sum(np.asarray(w.values) != ref))
        types.append(type(w).__name__)
        buf = w._buf.copy()
        buf[w._core()] = 0.0
        frame = max(frame, float(np.abs(buf).max()))
        contiguous = bool(w.values.flags.c_contiguous)
        v = w
    out.append([list(cells), corr.steps_per_period, mis, frame, types, contiguous, launches, list(ctx.plan())])
    wh.release_device_cache()
print(json.dumps(out))
"""


def test_seam_with_ghost_padded_fields(gpu_available):
    cases = [((300, 200), 21.0), ((40, 100, 130), 12.0), ((36, 61, 70), 11.0)]
    e = dict(os.environ, WHB_T3="1", WHB_PIPE="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT, "cases": cases}], capture_output=True, text=True,
                       env=e, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for cells, nt, mis, frame, types, contiguous, launches, plan in res:
        assert mis == 0, (cells, nt, launches, plan)
        assert frame == 0.0 and types == ["PaddedField"] * 2 and not contiguous, (cells, frame, types, contiguous)
        if len(cells) == 3:  # banded: one launch per pass and band
            assert plan[1] == 3 and min(launches) >= 2 * ((nt + 2) // 3), (cells, launches, plan)
