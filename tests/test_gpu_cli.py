"""GPU: paper_2504_03074_b200.cli converge (the reference's experiment runner, cli.py:252-331,
on the device solvers) against the CSVs the reference runner itself wrote for the same
arguments (tests/golden/cli/*, tests/golden/make_golden_cli.py): same config.txt and
config_hash line, same headers, same iteration counts and convergence flags, residual histories
to 1e-9 relative (explicit FPI iterates are bitwise; implicit inner CG and GMRES reductions are
not BLAS-ordered), predicted rate identical, measured rates to 1e-8.  Timing columns excluded
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
    c1, h1, r1 = read_csv(out / "residuals.csv")
    c2, h2, r2 = read_csv(os.path.join(GOLD, name, "residuals.csv"))
    assert c1 == c2 and h1 == h2 and len(r1) == len(r2)
    for a, b in zip(r1, r2):
        assert a[0] == b[0]
        for x, y in zip(a[1:], b[1:]):
            assert close(x, y, 1e-9), (name, a[0], x, y)
    c1, h1, s1 = read_csv(out / "summary.csv")
    c2, h2, s2 = read_csv(os.path.join(GOLD, name, "summary.csv"))
    assert c1 == c2 and h1 == h2
    for a, b in zip(s1, s2):
        for col, x, y in zip(h1, a, b):
            if "wall" in col or "seconds" in col:
                continue
            if col in ("method", "iterations", "converged", "predicted_mu"):
                assert x == y, (name, col, x, y)
            else:
                assert close(x, y, 1e-8) or (x == y == "nan"), (name, col, x, y)
