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
         ((128, 128), 20.3), ((100, 37), 25.0), ((5, 300), 9.0), ((37, 4), 3.0),
         # 3D, N_t mod 3 = 1 / 1 / 2 (three-step passes + a single / pair remainder), ragged tiles
         ((130, 70, 33), 25.0), ((40, 100, 130), 17.0), ((33, 33, 33), 14.0), ((48, 30, 200), 8.0)]

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
                                 {"WHB_T3": "1", "WHB_CHUNK3": "7"}, {"WHB_T3": "1", "WHB_CHUNK3": "1"},
                                 {"WHB_T3": "1", "WHB_CHUNK3": "500"}, {"WHB_T3": "0"},
                                 {"WHB_T3": "1", "WHB_T3_EDGE": "0"},
                                 {"WHB_KERNEL": "simple"}, {"WHB_NO_GRAPHS": "1"}])
def test_every_kernel_path_bitwise(gpu_available, env):
    e = dict(os.environ, **env)
    code = SCRIPT % {"root": ROOT, "cases": CASES}
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=e, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for cells, nt, mismatches, plan in res:
        assert mismatches == 0, (env, cells, nt, plan)
    if env.get("WHB_T3") == "1":  # the three-step kernel really ran on every 3D case
        assert all(p[1] == 3 for c, _, _, p in res if len(c) == 3), res
    # the default plan really uses the multi-step kernels
    if not env:
        plans = {tuple(c): tuple(p) for c, _, _, p in res}
        assert plans[(512, 512)][1] == 4 and plans[(64, 64, 64)] == (2, 2)
        # small 2D grids run cluster-resident (kernel 4)
        assert plans[(128, 128)][0] == 4 and plans[(256, 256)][0] == 4 and plans[(300, 300)][0] == 1


T3_SCRIPT = r"""
import json, sys, numpy as np
sys.path.insert(0, %(root)r)
import paper_2504_03074_b200 as wh
from paper_2504_03074_b200 import timestep as ts
from oracle import native as ON, waveholtz_oracle as O
ts._COURANT[2] = 0.9
out = []
# (cells, bounds, c, omega): square cells c = 1 (GM 2), c != 1 (GM 1), unequal spacing (GM 0)
for cells, hi, c, omega in [((40, 36, 44), (1.0, 1.0, 1.0), 1.0, 9.0), ((40, 36, 44), (1.0, 1.0, 1.0), 1.3, 9.0),
                            ((32, 50, 70), (1.0, 1.5, 2.0), 1.0, 6.0)]:
    g = wh.build_grid(3, [(0.0, h) for h in hi], list(cells), "dirichlet")
    f = wh.multi_gaussian_source(g, omega, 3, seed=2)
    fv = np.array(f.values)
    corr = wh.correct_explicit(omega, g, 2, c)
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    prob = wh.HelmholtzProblem(g, 2, c, omega, f)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    v, run = wh.fpi_solve(prob, cfg, tol=-1.0, maxit=3)
    vref, rref = ON.fpi(fv, g.spacing, sc, 3, c=c)
    x = np.random.default_rng(3).standard_normal(g.shape) * 1e-2
    x = np.array(wh.GridField.from_values(g, x).values)
    av = wh.waveholtz_operator(prob, cfg, corr=corr)(x)
    avref = x - ON.wave_solve(x, None, g.spacing, sc, c=c, zero_f=True)
    dp = wh.device.device_problem(g, c=c)
    out.append([list(cells), c, corr.steps_per_period, int(np.sum(v.values != vref)),
                max(abs(a - b) / b for a, b in zip(run.residuals, rref)), int(np.sum(av != avref)),
                list(dp.ctx.plan())])
    wh.release_device_cache()
print(json.dumps(out))
"""


def test_three_step_kernel_fpi_matvec_geometry_modes(gpu_available):
    """The three-step 3D kernel (forced on small grids, chunked) in FPI mode (residual fused in the
    last pass) and as the GMRES mat-vec (zero forcing, x - W(x, 0)), for the three geometry modes:
    iterates and A x bitwise equal to the C restatement, residuals to 1e-12."""
    e = dict(os.environ, WHB_T3="1", WHB_CHUNK3="9")
    r = subprocess.run([sys.executable, "-c", T3_SCRIPT % {"root": ROOT}], capture_output=True, text=True, env=e,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    for cells, c, nt, vmis, rerr, avmis, plan in json.loads(r.stdout.strip().splitlines()[-1]):
        assert plan[1] == 3, plan
        assert vmis == 0 and avmis == 0 and rerr <= 1e-12, (cells, c, nt, vmis, avmis, rerr)


BAND_SCRIPT = r"""
import json, sys, numpy as np
sys.path.insert(0, %(root)r)
import paper_2504_03074_b200 as wh
from paper_2504_03074_b200 import timestep as ts
from oracle import native as ON, waveholtz_oracle as O
ts._COURANT[2] = 0.9
out = []
# N_t mod 3 = 0 / 1 / 2 (last pass: three-step kernel / two two-step passes / one two-step pass)
for cells, omega in [((40, 100, 130), 12.0), ((48, 30, 200), 8.0), ((64, 64, 64), 11.0), ((33, 50, 33), 13.0),
                     ((36, 61, 70), 11.0)]:
    g = wh.build_grid(3, [(0.0, 1.0)] * 3, list(cells), "dirichlet")
    f = wh.multi_gaussian_source(g, omega, 3, seed=4)
    corr = wh.correct_explicit(omega, g, 2, 1.0)
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    prob = wh.HelmholtzProblem(g, 2, 1.0, omega, f)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    step = wh.HostFPIStep(prob, cfg)
    rng = np.random.default_rng(5)
    a = rng.standard_normal(g.shape) * 1e-3      # nonzero boundary values: the upload must zero them
    b = np.full(g.shape, np.nan)
    ref = np.array(wh.GridField.from_values(g, a).values)
    mis, rerr, launches = 0, 0.0, []
    for it in range(3):
        l0 = step.dp.ctx.launch_count()
        d = step(a, b)
        launches.append(step.dp.ctx.launch_count() - l0)
        new = ON.wave_solve(ref, np.array(f.values), g.spacing, sc)
        dref = float(np.sqrt(np.sum((new - ref) ** 2)) / np.sqrt(g.size))
        mis += int(np.sum(b != new))
        rerr = max(rerr, abs(d - dref) / dref)
        ref = new
        a, b = b, a      # feed the iterate back (the reference's _iterate loop)
    # the Python seam (host GridField in, new GridField out: whb_solve_host, plain output), twice
    op = wh.DiscreteOperator(g, 2, 1.0)
    vf = wh.GridField.from_values(g, rng.standard_normal(g.shape) * 1e-3)
    for it in range(2):
        l0 = step.dp.ctx.launch_count()
        wf = wh.wave_solve_filtered(vf, f, cfg, corr, op)
        launches.append(step.dp.ctx.launch_count() - l0)
        mis += int(np.sum(wf.values != ON.wave_solve(np.array(vf.values), np.array(f.values), g.spacing, sc)))
        vf = wf
    out.append([list(cells), corr.steps_per_period, mis, rerr, launches, list(step.dp.ctx.plan())])
    wh.release_device_cache()
print(json.dumps(out))
"""


@pytest.mark.parametrize("env", [{}, {"WHB_PIPE_ROWS": "3"}, {"WHB_PIPE": "0"}, {"WHB_T3_EDGE": "0"}])
def test_banded_host_iteration_bitwise(gpu_available, env):
    """whb_iterate_host on the three-step plan hides the host transfers behind (pass, row band)
    launches enqueued by diagonals: v_new bitwise equal to the C restatement for 3 chained
    iterations (every remainder of N_t mod 3, ragged bands, every edge tile shape), the residual
    to 1e-12; WHB_PIPE=0 is the serial path."""
    e = dict(os.environ, WHB_T3="1", **{"WHB_PIPE": "1", **env})  # WHB_PIPE=1: bands on small grids too
    r = subprocess.run([sys.executable, "-c", BAND_SCRIPT % {"root": ROOT}], capture_output=True, text=True, env=e,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert {nt % 3 for _, nt, *_ in res} == {0, 1, 2}, res
    banded = 0
    for cells, nt, mis, rerr, launches, plan in res:
        assert plan[1] == 3, plan
        assert mis == 0, (env, cells, nt, launches)
        assert rerr < 1e-12, (env, cells, rerr)
        passes = (nt + 2) // 3
        if env.get("WHB_PIPE") == "0":
            assert max(launches) < 2 * passes, launches
        banded += min(launches) >= 2 * passes  # one launch per pass and band (>= 2 bands)
    if env.get("WHB_PIPE") != "0":  # the banded path really ran (grids of one band keep the serial path)
        assert banded >= (3 if "WHB_PIPE_ROWS" in env else 5), res
