"""GPU: slab-decomposed solves (several whb contexts owning axis-0 plane ranges,
region-split steps, ghost-plane copies) equal the single-domain reference
iterates bitwise.  Runs all slabs in one process on one GPU (LocalHalo); the
cross-rank driver is covered on CPU by tests/test_slab_gloo.py."""

import numpy as np
import pytest

import paper_2504_03074_b200 as wh
from paper_2504_03074_b200 import _native
from paper_2504_03074_b200.slab import DeviceShard, LocalHalo, run_local_solve, slab_ranges
from oracle import native as ON
from oracle import waveholtz_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cells,nslabs,omega", [((69, 49), 4, 15.0), ((32, 19, 23), 3, 9.0), ((8, 12, 10), 4, 5.0),
                                                ((64, 64, 64), 2, 20.0)])
def test_local_slabs_match_single_domain_bitwise(gpu_available, cells, nslabs, omega):
    d = len(cells)
    g = wh.build_grid(d, [(0.0, 1.0)] * d, cells, "dirichlet")
    f = O.multi_gaussian(g.shape, g.bounds, g.spacing, 3, seed=2)
    corr = wh.correct_explicit(omega, g, 2, 1.0)
    cfg = wh.FilterConfig(omega=omega, periods=1, steps_per_period=corr.steps_per_period, mode="explicit")
    sched = wh.time_schedule(corr, cfg)
    ranges = slab_ranges(g.shape[0], nslabs)
    shards = [DeviceShard(g, r) for r in ranges]
    for sh, (p0, p1) in zip(shards, ranges):
        sh.set_schedule(sched)
        sh.upload(_native.F, np.ascontiguousarray(f[p0:p1]))
        sh.zero(_native.V)
    halo = LocalHalo(shards)
    iters = 3
    sums = [sum(run_local_solve(shards, halo)) for _ in range(iters)]
    for sh in shards:
        sh.synchronize()
    v = np.concatenate([sh.download(_native.V) for sh in shards], axis=0)
    sc = O.step_scalars(corr.steps_per_period, corr.dt, corr.omega_tilde)
    vref, rref = ON.fpi(f, g.spacing, sc, iters)
    assert np.array_equal(v, vref)
    np.testing.assert_allclose(np.sqrt(sums) / np.sqrt(g.size), rref, rtol=1e-12)
