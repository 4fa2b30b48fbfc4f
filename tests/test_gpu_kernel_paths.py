"""GPU: every selectable kernel path (launch plan) gives the reference's bits.

The default plan picks the 2D wavefront kernel (4 or 2 steps per pass), the
two-step kernel (3D) and the one-step TMA/bulk kernels for remainders and
slabs; WHB_* environment switches force the others.  Sizes are chosen so the
march is chunked (halo rows shared between CTAs), the step count leaves every
remainder mod 4, and grids are ragged with respect to the tiles."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

CASES = [((512, 512), 40.0), ((512, 512), 61.0), ((1024, 1024), 90.0), ((600, 600), 50.0), ((300, 300), 33.0),
         ((256, 256), 40.0), ((400, 250), 30.0), ((90, 47, 61), 20.0), ((64, 64, 64), 11.0),
         ((128, 128), 20.3), ((100, 37), 25.0), ((5, 300), 9.0), ((37, 4), 3.0)]

SCRIPT = r"""
import json, sys, numpy as np
sys.path.insert(0, %(root)r)
import paper_2504_03074_b200 as wh
from paper_2504_03074_b200 import timestep as ts
from oracle import native as ON, waveholtz_oracle as O
ts._COURANT[2] = 0.9
out = []
for cells, omega in %(cases)r:
    d = len(cells)
    g = wh.build_grid(d, [(0.0, 1.0)] * d, list(cells), "dirichlet")
    f = wh.multi_gaussian_source(g, omega, 4, seed=1)
    v = wh.GridField.from_values(g, np.random.default_rng(11).standard_normal(g.shape) * 1e-3)
    corr = wh.correct_explicit(omega, g, 2, 1.0)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    got = wh.wave_solve_filtered(v, f, cfg, corr, wh.DiscreteOperator(g, 2, 1.0)).values
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    ref = ON.wave_solve(np.array(v.values), np.array(f.values), g.spacing, sc)
    dp = wh.device.device_problem(g)
    out.append([list(cells), corr.steps_per_period, int(np.sum(got != ref)), list(dp.ctx.plan())])
    wh.release_device_cache()
print(json.dumps(out))
"""


@pytest.mark.parametrize("env", [{}, {"WHB_CRES": "0"}, {"WHB_CRES_CL": "8"}, {"WHB_CRES_CL": "3"}, {"WHB_WF": "2"}, {"WHB_WF": "0"}, {"WHB_TB2": "0"}, {"WHB_KERNEL": "bulk"},
                                 {"WHB_KERNEL": "simple"}, {"WHB_NO_GRAPHS": "1"}])
def test_every_kernel_path_bitwise(gpu_available, env):
    e = dict(os.environ, **env)
    code = SCRIPT % {"root": ROOT, "cases": CASES}
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=e, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for cells, nt, mismatches, plan in res:
        assert mismatches == 0, (env, cells, nt, plan)
    # the default plan really uses the multi-step kernels
    if not env:
        plans = {tuple(c): tuple(p) for c, _, _, p in res}
        assert plans[(512, 512)][1] == 4 and plans[(64, 64, 64)] == (2, 2)
        # small 2D grids run cluster-resident (kernel 4)
        assert plans[(128, 128)][0] == 4 and plans[(256, 256)][0] == 4 and plans[(300, 300)][0] == 1
