"""CPU: pin the implicit-path oracle restatement (oracle/implicit_oracle.py)
against golden outputs of the reference itself (tests/golden/implicit.*)."""

import json
import math
import os

import numpy as np
import pytest

from conftest import ROOT
from oracle import implicit_oracle as IO

GOLD = os.path.join(ROOT, "tests", "golden")
META = json.load(open(os.path.join(GOLD, "implicit.json")))
ARR = np.load(os.path.join(GOLD, "implicit.npz"))


def spacing(m):
    return tuple(1.0 / n for n in m["cells"])


@pytest.mark.parametrize("name", sorted(META))
def test_oracle_implicit_wave_solve_bitwise(name):
    m = META[name]
    bcs = [m["bcs"]] * m["dim"]
    out, solver = IO.wave_solve_implicit(ARR[f"{name}/v0"], ARR[f"{name}/f"], spacing(m), bcs, m["order"],
                                         m["omega"], m["n_t"], implicit_first_step=m["implicit_first_step"])
    assert np.array_equal(out, ARR[f"{name}/out"])
    assert solver.inner == m["inner"]


@pytest.mark.parametrize("name", [n for n in sorted(META) if "fpi_residuals" in META[n]])
def test_oracle_implicit_fpi(name):
    m = META[name]
    bcs = [m["bcs"]] * m["dim"]
    f = ARR[f"{name}/f"]
    v = np.zeros_like(f)
    solver = None
    res = []
    for k in range(len(m["fpi_residuals"])):
        v_new, solver = IO.wave_solve_implicit(v, f, spacing(m), bcs, m["order"], m["omega"], m["n_t"],
                                               solver=solver)
        res.append(float(np.linalg.norm(v_new - v) / math.sqrt(v.size)))
        v = v_new
        assert np.array_equal(v, ARR[f"{name}/fpi{k + 1}"])
    assert res == m["fpi_residuals"]


def test_correct_implicit_matches_reference_formula():
    n_t, dt, wi = IO.correct_implicit(5.5, 10)
    assert n_t == 10 and abs(math.cos(wi * dt) * (1.0 + (5.5 * dt) ** 2 / 2.0) - 1.0) <= 1e-13
    with pytest.raises(ValueError):
        IO.correct_implicit(5.5, 4)
