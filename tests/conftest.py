"""Shared test helpers.  `-m gpu` tests need a CUDA device (run through gpurun);
everything else runs on the CPU-only build container."""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


def sha(a) -> str:
    """sha256 of the C-order float64 bytes (hashed in place: no copy of a 8.6 GB iterate)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    return hashlib.sha256(a.data if a.flags.c_contiguous else a.tobytes()).hexdigest()


def load_golden(name):
    path = os.path.join(GOLDEN, f"{name}.json")
    if not os.path.exists(path):
        pytest.fail(f"golden fixture {name} missing (tests/golden/make_golden.py {name})")
    meta = json.load(open(path))
    npz = os.path.join(GOLDEN, f"{name}.npz")
    arrays = np.load(npz) if os.path.exists(npz) else None
    return meta, arrays


def spacing_of(case):
    return tuple((hi - lo) / n for (lo, hi), n in zip(case["bounds"], case["cells"]))


def rel_maxnorm(a, b):
    scale = float(np.max(np.abs(b)))
    return float(np.max(np.abs(a - b))) / (scale if scale > 0 else 1.0)


@pytest.fixture(scope="session")
def gpu_available():
    from paper_2504_03074_b200 import _native

    if _native.device_count() < 1:
        pytest.fail("a -m gpu test ran without a CUDA device")
    return True
