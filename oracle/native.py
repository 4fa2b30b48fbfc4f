"""TEST INFRASTRUCTURE ONLY — ctypes loader for the C restatement (oracle/whb_oracle.c).

Used by tests/ (parity checker at sizes numpy is too slow for) and bench.py
(multi-core CPU baseline).  The product package never imports it.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libwhb_oracle.so")

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        L.who_wave_solve.argtypes = [ctypes.c_int, ip, dp, dp, ctypes.c_double, dp, dp, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_double, ctypes.c_double, dp, dp,
                                     ctypes.c_double, dp, ctypes.c_int]
        L.who_fpi.argtypes = [ctypes.c_int, ip, dp, dp, ctypes.c_double, dp, ctypes.c_int,
                              ctypes.c_double, ctypes.c_double, dp, dp, ctypes.c_double, ctypes.c_int,
                              dp, dp, ctypes.c_int]
        L.who_fpi_lean.argtypes = L.who_fpi.argtypes + [ctypes.c_int]
        L.who_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _coeffs(spacing, c):
    """Host scalars exactly as the reference forms them (grid.py:302-306, 366)."""
    clo = np.array([(np.array([1.0, -2.0, 1.0]) / dx**2)[0] for dx in spacing])
    cmid = np.array([(np.array([1.0, -2.0, 1.0]) / dx**2)[1] for dx in spacing])
    return clo, cmid, float(c**2)


def max_threads() -> int:
    return lib().who_max_threads()


def auto_threads(npoints: int) -> int:
    """One thread per ~256K points (tiny grids stay serial: no per-step fork/join)."""
    return max(1, min(max_threads(), npoints // 262144))


def wave_solve(v, f, spacing, sc, c=1.0, zero_f=False, nthreads=0):
    v = np.ascontiguousarray(v, dtype=np.float64)
    f = np.ascontiguousarray(f if f is not None else np.zeros_like(v), dtype=np.float64)
    shape = np.array(v.shape, dtype=np.int64)
    clo, cmid, c2 = _coeffs(spacing, c)
    cos_f = np.ascontiguousarray(sc["cos_f"], dtype=np.float64)
    acc_c = np.ascontiguousarray(sc["acc_c"], dtype=np.float64)
    out = np.empty_like(v)
    rc = lib().who_wave_solve(v.ndim, shape.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dp(clo),
                              _dp(cmid), c2, _dp(v), _dp(f), int(zero_f), sc["n_total"], sc["half_dt2"],
                              sc["dt2"], _dp(cos_f), _dp(acc_c), sc["out_scale"], _dp(out),
                              nthreads or auto_threads(v.size))
    if rc:
        raise RuntimeError(f"who_wave_solve rc={rc}")
    return out


def fpi(f, spacing, sc, iters, c=1.0, nthreads=0):
    f = np.ascontiguousarray(f, dtype=np.float64)
    shape = np.array(f.shape, dtype=np.int64)
    clo, cmid, c2 = _coeffs(spacing, c)
    cos_f = np.ascontiguousarray(sc["cos_f"], dtype=np.float64)
    acc_c = np.ascontiguousarray(sc["acc_c"], dtype=np.float64)
    v = np.empty_like(f)
    res = np.empty(iters)
    rc = lib().who_fpi(f.ndim, shape.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dp(clo), _dp(cmid),
                       c2, _dp(f), sc["n_total"], sc["half_dt2"], sc["dt2"], _dp(cos_f), _dp(acc_c),
                       sc["out_scale"], iters, _dp(v), _dp(res), nthreads or auto_threads(f.size))
    if rc:
        raise RuntimeError(f"who_fpi rc={rc}")
    return v, list(res)


def fpi_lean(f, spacing, sc, iters, c=1.0, nthreads=0, v=None):
    """fpi() with 5 resident fields instead of 8 (for 1025^3 on a 62 GB host); bitwise the same.
    ``v`` (C-contiguous float64, updated in place) continues from a previous iterate."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    shape = np.array(f.shape, dtype=np.int64)
    clo, cmid, c2 = _coeffs(spacing, c)
    cos_f = np.ascontiguousarray(sc["cos_f"], dtype=np.float64)
    acc_c = np.ascontiguousarray(sc["acc_c"], dtype=np.float64)
    given = v is not None
    if given:
        assert v.dtype == np.float64 and v.flags.c_contiguous and v.shape == f.shape
    else:
        v = np.empty_like(f)
    res = np.empty(iters)
    rc = lib().who_fpi_lean(f.ndim, shape.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dp(clo), _dp(cmid),
                            c2, _dp(f), sc["n_total"], sc["half_dt2"], sc["dt2"], _dp(cos_f), _dp(acc_c),
                            sc["out_scale"], iters, _dp(v), _dp(res), nthreads or auto_threads(f.size),
                            int(given))
    if rc:
        raise RuntimeError(f"who_fpi_lean rc={rc}")
    return v, list(res)
