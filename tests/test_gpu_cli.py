"""GPU: paper_2504_03074_b200.cli converge (the reference's experiment runner, cli.py:252-331,
on the device solvers) against the CSVs the reference runner itself wrote for the same
arguments (tests/golden/cli/*, tests/golden/make_golden_cli.py): same config.txt and
config_hash line, same headers, same iteration counts and convergence flags, predicted rate
identical.  Residual histories and measured rates: 1e-9 relative in explicit mode (the iterates are
bitwise; only the norms' summation order differs); 1e-6 in implicit mode, where iterates agree to
the inner CG tolerance (1e-12 relative, about 1e-10 of the iterate) and a residual
||v_k+1 - v_k|| of 1e-8 is a difference of nearly equal iterates.  Timing columns excluded
(cli.py:5-7)."""

import csv
import os

import pytest

from conftest import ROOT
from test_cli_cpu import CASES

from paper_2504_03074_b200 import cli

pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden", "cli")


def read_csv(path):
    lines = open(path).read().splitlines()
    rows = list(csv.reader(lines[1:]))
    return lines[0], rows[0], rows[1:]


def close(a, b, rtol):
    if a == b:
        return True
    if a == "" or b == "" or a == "nan" or b == "nan":
        return False
    x, y = float(a), float(b)
    return abs(x - y) <= rtol * max(abs(x), abs(y))


@pytest.mark.parametrize("name", sorted(CASES))
def test_converge_matches_reference_runner(gpu_available, name, tmp_path):
    out = tmp_path / name
    assert cli.main(CASES[name] + ["--out", str(out)]) == 0
    assert (out / "config.txt").read_text() == open(os.path.join(GOLD, name, "config.txt")).read()
    rtol = 1e-6 if "implicit" in name else 1e-9
    c1, h1, r1 = read_csv(out / "residuals.csv")
    c2, h2, r2 = read_csv(os.path.join(GOLD, name, "residuals.csv"))
    assert c1 == c2 and h1 == h2 and len(r1) == len(r2)
    for a, b in zip(r1, r2):
        assert a[0] == b[0]
        for x, y in zip(a[1:], b[1:]):
            assert close(x, y, rtol), (name, a[0], x, y)
    c1, h1, s1 = read_csv(out / "summary.csv")
    c2, h2, s2 = read_csv(os.path.join(GOLD, name, "summary.csv"))
    assert c1 == c2 and h1 == h2
    for a, b in zip(s1, s2):
        for col, x, y in zip(h1, a, b):
            if "wall" in col or "seconds" in col:
                continue
            if col in ("method", "iterations", "converged", "predicted_mu"):
                assert x == y, (name, col, x, y)
            elif col == "relative_gap":  # |cr - mu| / mu of two nearly equal rates: absolute
                assert x == y == "nan" or abs(float(x) - float(y)) <= max(rtol, 1e-8), (name, col, x, y)
            else:
                assert close(x, y, max(rtol, 1e-8)) or (x == y == "nan"), (name, col, x, y)
