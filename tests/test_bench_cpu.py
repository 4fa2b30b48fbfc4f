"""CPU: bench.py's reference arm runs here (it times the bitwise C restatement of the
reference on the host cores) and prints one JSON line with the contract's keys."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


@pytest.mark.parametrize("workload", ["cfg1", "cfg2"])
def test_reference_arm_json_line(workload):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", workload,
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"]["workload"] == workload
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1


def test_gpus_n_self_launches_slab_ranks_gloo():
    """bench.py --gpus 2 without torchrun re-launches itself through torch.distributed.run: two
    ranks run the z-slab driver (slab.SlabFPI + TorchHalo) over gloo with the numpy stand-in
    shard, rank 0 prints ONE line with n_gpus 2, the z-slab parallelism and strong scaling, and the
    residuals equal the single-domain oracle's (the decomposition really ran)."""
    import numpy as np

    from oracle import waveholtz_oracle as O
    import paper_2504_03074_b200 as wh
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", "cfg3",
                        "--cells", "20", "--steps", "2", "--warmup", "1", "--emulate-cpu"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["parallelism"].startswith("z-slab decomposition over 2 GPUs")
    assert line["config"]["grid"] == [21, 21, 21] and line["config"]["N_t"] > 0
    # residuals of the 2 timed iterations (from v = 0) against the single-domain oracle
    g = wh.build_grid(3, [(0.0, 1.0)] * 3, [20] * 3, "dirichlet")
    f = np.array(wh.gaussian_source(g, 40.7, 100.0, 300.0, (0.45, 0.5, 0.55)).values)
    n_t, dt, we = O.correct_explicit(40.7, g.spacing, 2, 1.0, 0.9)
    _, rref = O.fpi(f, g.spacing, O.step_scalars(n_t, dt, we), 2)
    assert abs(line["residuals"]["first"] - rref[0]) <= 1e-12 * rref[0]
    assert abs(line["residuals"]["last"] - rref[1]) <= 1e-12 * rref[1]
