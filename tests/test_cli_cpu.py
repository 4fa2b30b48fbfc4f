"""CPU: the host half of paper_2504_03074_b200.cli (config parsing, config_hash, CSV format,
exit codes) and the rate prediction it prints (rates.py) against the reference runner's own
outputs (tests/golden/cli/*, made by tests/golden/make_golden_cli.py) and, where the reference is
importable here, against its filter theory directly."""

import csv
import math
import os

import numpy as np
import pytest

from conftest import ROOT

import paper_2504_03074_b200 as wh
from paper_2504_03074_b200 import cli
from paper_2504_03074_b200.rates import discrete_eigenvalues_symbolic, predict_rate

GOLD = os.path.join(ROOT, "tests", "golden", "cli")
CASES = {
    "explicit_2d": ["converge", "--mode", "explicit", "--dim", "2", "--cells", "48", "--omega", "9.3",
                    "--center", "0.4,0.6", "--width", "60", "--tol", "1e-8", "--maxit", "400"],
    "explicit_1d_p4": ["converge", "--mode", "explicit", "--cells", "40", "--order", "4", "--omega", "7.1",
                       "--tol", "1e-9", "--maxit", "500"],
    "implicit_1d": ["converge", "--cells", "32", "--tol", "1e-10"],
    "implicit_2d": ["converge", "--dim", "2", "--cells", "32", "--omega", "6.2", "--center", "0.45,0.55",
                    "--nt", "12", "--tol", "1e-9", "--maxit", "300"],
}


def read_csv(path):
    lines = open(path).read().splitlines()
    rows = list(csv.reader(lines[1:]))
    return lines[0], rows[0], rows[1:]


def effective_cfg(args):
    cfg = dict(cli._DEFAULTS[args[0]])
    cfg.update(cli._parse_overrides(args[1:]))
    return cfg


@pytest.mark.parametrize("name", sorted(CASES))
def test_config_text_hash_and_predicted_rate_match_reference_runner(name):
    cfg = effective_cfg(CASES[name])
    assert cli.canonical_text(cfg) == open(os.path.join(GOLD, name, "config.txt")).read()
    comment, header, rows = read_csv(os.path.join(GOLD, name, "summary.csv"))
    assert comment == f"# config_hash={cli.config_hash(cfg)}"
    # predicted_mu of the fixed point: discrete spectrum + filter theory on the host
    prob = cli._build_problem(cfg)
    config = wh.FilterConfig(omega=prob.omega, periods=int(cfg["periods"]), steps_per_period=int(cfg["nt"]),
                             mode=cfg["mode"])
    corr, cfg_eff = wh.resolve_time_discretization(prob, config)
    mu = predict_rate(discrete_eigenvalues_symbolic(prob.grid, prob.order, prob.c), cfg_eff,
                      omega_tilde=corr.omega_tilde).mu
    got = {r[0]: r for r in rows}
    assert cli._fmt(mu) == got["fpi"][header.index("predicted_mu")]


def test_csv_format_and_exit_codes(tmp_path):
    p = cli.write_csv(tmp_path / "x.csv", ["a", "b", "c"], [(1, 2.5, "z"), (True, np.float64(1e-3), "")], "abc")
    assert p.read_text() == "# config_hash=abc\na,b,c\n1,2.50000000000e+00,z\n1,1.00000000000e-03,\n"
    assert cli.main(["converge", "--nosuchkey", "1", "--out", str(tmp_path / "o")]) == 1
    assert cli.main(["converge", "--deflate", "2", "--out", str(tmp_path / "d")]) == 1
    assert cli.main(["converge", "--cells", "x", "--out", str(tmp_path / "e")]) == 1
    assert cli.main(["nosuchcommand"]) == 1


def test_rates_against_reference_filter_theory():
    from oracle import reference_harness as RH

    if not RH.available():
        pytest.skip("reference not importable (GPU box)")
    ref = RH.import_reference()
    import waveholtz.filters as F
    import waveholtz.grid as G

    for dim, cells, order, c, bcs in [(1, [37], 2, 1.0, "dirichlet"), (2, [24, 18], 4, 1.3, "dirichlet"),
                                      (2, [20, 16], 2, 1.0, "periodic"), (1, [33], 4, 0.7, "periodic")]:
        g = wh.build_grid(dim, [(0.0, 1.0)] * dim, cells, bcs)
        gr = G.build_grid(dim, [(0.0, 1.0)] * dim, cells, bcs)
        a = discrete_eigenvalues_symbolic(g, order, c)
        b = G.discrete_eigenvalues_symbolic(gr, order, c)
        assert np.array_equal(a, b)
        for mode, nt in (("explicit", 40), ("implicit", 12), ("continuous", 10)):
            cfg = wh.FilterConfig(omega=7.3, periods=2, steps_per_period=nt, mode=mode)
            cfr = F.FilterConfig(omega=7.3, periods=2, steps_per_period=nt, mode=mode)
            assert predict_rate(a, cfg, omega_tilde=7.31).mu == F.predict_rate(b, cfr, omega_tilde=7.31).mu
    del ref
