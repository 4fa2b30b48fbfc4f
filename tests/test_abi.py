"""CPU: the C-ABI library loads, exports every symbol include/whb200.h declares,
and the product path fails loudly (no CPU fallback) when no GPU is visible."""

import os
import re
import subprocess

import pytest

from conftest import ROOT

from paper_2504_03074_b200 import _native

HEADER = os.path.join(ROOT, "include", "whb200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(whb_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    syms = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    for name in declared():
        assert name in syms, name
        assert getattr(lib, name) is not None


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_no_device_behaviour():
    lib = _native.load()
    want = int(re.search(r"#define WHB_ABI_VERSION (\d+)", open(HEADER).read()).group(1))
    assert lib.whb_abi_version() == want
    if _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(_native.NativeError):
        _native.Context((9, 9))
    assert b"device" in lib.whb_last_error().lower()


def test_null_arguments_are_rejected():
    lib = _native.load()
    assert lib.whb_create(None, 0, 2, None, 0, 1, 1, 0) == _native.E_ARG
    assert lib.whb_destroy(None) == 0
    assert lib.whb_fpi(None, 1, -1.0, None, None) == _native.E_ARG
    assert lib.whb_fpi_scaled(None, 1, -1.0, 1.0, None, None) == _native.E_ARG


def test_context_binding_is_complete():
    """Every method the product modules call on a context exists on _native.Context (a module-level
    def placed inside the class once silently truncated it; this catches that on the CPU)."""
    import inspect
    import re as _re

    pkg = os.path.join(ROOT, "paper_2504_03074_b200")
    used = set()
    for fn in os.listdir(pkg):
        if fn.endswith(".py") and fn != "_native.py":
            used |= set(_re.findall(r"\bctx\.([a-z_][a-z0-9_]*)\(", open(os.path.join(pkg, fn)).read()))
    have = {n for n, _ in inspect.getmembers(_native.Context)}
    missing = sorted(used - have)
    assert not missing, missing
