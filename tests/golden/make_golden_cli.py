"""Golden CSVs of the reference's own experiment runner (``waveholtz.cli.main``, cli.py:541-591)
for the ``converge`` command, run in the build container where /root/reference exists:

    python tests/golden/make_golden_cli.py

writes tests/golden/cli/<case>/{config.txt, residuals.csv, summary.csv}.  The GPU test
(tests/test_gpu_cli.py) runs paper_2504_03074_b200.cli with the same arguments and compares."""

import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import reference_harness as RH  # noqa: E402

CASES = {
    "explicit_2d": ["converge", "--mode", "explicit", "--dim", "2", "--cells", "48", "--omega", "9.3",
                    "--center", "0.4,0.6", "--width", "60", "--tol", "1e-8", "--maxit", "400"],
    "explicit_1d_p4": ["converge", "--mode", "explicit", "--cells", "40", "--order", "4", "--omega", "7.1",
                       "--tol", "1e-9", "--maxit", "500"],
    "implicit_1d": ["converge", "--cells", "32", "--tol", "1e-10"],
    "implicit_2d": ["converge", "--dim", "2", "--cells", "32", "--omega", "6.2", "--center", "0.45,0.55",
                    "--nt", "12", "--tol", "1e-9", "--maxit", "300"],
}


def main():
    wh = RH.import_reference()
    import waveholtz.cli as cli

    for name, args in CASES.items():
        out = os.path.join(HERE, "cli", name)
        shutil.rmtree(out, ignore_errors=True)
        rc = cli.main(args + ["--out", out])
        assert rc == 0, (name, rc)
        print(name, "ok", flush=True)
    del wh


if __name__ == "__main__":
    main()
