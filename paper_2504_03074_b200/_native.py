"""ctypes binding of the C ABI in include/whb200.h (libwhb200.so, sm_100a).

This is the only path to compute: there is no CPU fallback.  If the library
is missing or no CUDA device is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libwhb200.so")
# tuning sweeps only: WHB_LIB names a variant build under lib/variants/ (tools/variants.py)
if os.environ.get("WHB_LIB"):
    LIB_PATH = os.path.join(_PKG, "lib", "variants", os.path.basename(os.environ["WHB_LIB"]))

# enum whb_field / whb_out_mode (include/whb200.h)
V, F, WA, WB, ACC, OUT, WC, WD = range(8)
OUT_PLAIN, OUT_FPI, OUT_AV = 0, 1, 2
E_ARG, E_CUDA, E_NOMEM, E_STATE, E_NODEV = -1, -2, -3, -4, -5

#: every symbol include/whb200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "whb_abi_version", "whb_last_error", "whb_device_count", "whb_create", "whb_destroy",
    "whb_set_operator", "whb_set_schedule", "whb_upload", "whb_download", "whb_zero",
    "whb_filtered_solve", "whb_fpi", "whb_fpi_scaled", "whb_ipc_handle", "whb_ipc_open", "whb_ipc_close",
    "whb_flags_alloc", "whb_flags_free", "whb_copy_async", "whb_stream_write_u32", "whb_stream_wait_u32",
    "whb_capture_begin", "whb_capture_end", "whb_graph_launch", "whb_resid_read", "whb_iterate_host", "whb_vec_reserve", "whb_vec_upload",
    "whb_vec_download", "whb_vec_dot", "whb_vec_axpy", "whb_vec_scale_into", "whb_vec_div_into",
    "whb_vec_lincomb", "whb_vec_sub_into", "whb_vec_copy", "whb_matvec", "whb_solve_begin",
    "whb_step", "whb_solve_end", "whb_level_plane_ptr", "whb_stream_ptr", "whb_synchronize",
    "whb_copy_plane", "whb_launch_count", "whb_set_timing", "whb_last_timing", "whb_host_alloc",
    "whb_host_free", "whb_geometry", "whb_set_l2_flush", "whb_apply_operator", "whb_plan", "whb_set_operator_general",
    "whb_pair", "whb_triple", "whb_ghost_planes", "whb_field_plane_ptr", "whb_copy_device",
    "whb_imp_apply", "whb_imp_rhs", "whb_vec_xpay", "whb_mg_setup", "whb_mg_vcycle", "whb_tri_setup", "whb_tri_solve",
    "whb_cg_begin", "whb_cg_iterate", "whb_vec_mgs",
    "whb_comm_begin", "whb_comm_end", "whb_comm_join", "whb_nccl_unique_id", "whb_nccl_init", "whb_nccl_exchange",
    "whb_nccl_allreduce_sum", "whb_upload_strided", "whb_download_strided", "whb_solve_host",
)

_lib = None


class NativeError(RuntimeError):
    """A whb_* call failed on the device side."""


def load():
    """Load libwhb200.so (fails loudly when the extension was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    c_int, c_double, c_i64, c_u64 = ctypes.c_int, ctypes.c_double, ctypes.c_int64, ctypes.c_uint64
    vp, dp, ip64 = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
    sig = {
        "whb_abi_version": ([], c_int),
        "whb_last_error": ([], ctypes.c_char_p),
        "whb_device_count": ([ctypes.POINTER(c_int)], c_int),
        "whb_create": ([ctypes.POINTER(vp), c_int, c_int, ip64, c_i64, c_i64, c_int, c_int], c_int),
        "whb_destroy": ([vp], c_int),
        "whb_set_operator": ([vp, dp, dp, c_double], c_int),
        "whb_set_schedule": ([vp, c_int, c_int, c_double, c_double, dp, dp, c_double], c_int),
        "whb_upload": ([vp, c_int, c_int, dp], c_int),
        "whb_download": ([vp, c_int, c_int, dp], c_int),
        "whb_zero": ([vp, c_int, c_int], c_int),
        "whb_filtered_solve": ([vp, c_int, c_int, dp], c_int),
        "whb_fpi": ([vp, c_int, c_double, dp, ctypes.POINTER(c_int)], c_int),
        "whb_fpi_scaled": ([vp, c_int, c_double, c_double, dp, ctypes.POINTER(c_int)], c_int),
        "whb_ipc_handle": ([vp, c_u64, ctypes.c_char_p, ip64], c_int),
        "whb_ipc_open": ([vp, ctypes.c_char_p, ctypes.POINTER(c_u64)], c_int),
        "whb_ipc_close": ([vp, c_u64], c_int),
        "whb_flags_alloc": ([vp, c_int, ctypes.POINTER(c_u64)], c_int),
        "whb_flags_free": ([vp, c_u64], c_int),
        "whb_copy_async": ([vp, c_u64, c_u64, c_i64], c_int),
        "whb_capture_begin": ([vp], c_int),
        "whb_capture_end": ([vp, ctypes.POINTER(c_int)], c_int),
        "whb_graph_launch": ([vp, c_int], c_int),
        "whb_resid_read": ([vp, dp], c_int),
        "whb_stream_write_u32": ([vp, c_u64, ctypes.c_uint32], c_int),
        "whb_stream_wait_u32": ([vp, c_u64, ctypes.c_uint32], c_int),
        "whb_upload_strided": ([vp, c_int, c_int, dp, c_i64, c_i64], c_int),
        "whb_download_strided": ([vp, c_int, c_int, dp, c_i64, c_i64], c_int),
        "whb_comm_begin": ([vp], c_int),
        "whb_comm_end": ([vp], c_int),
        "whb_comm_join": ([vp], c_int),
        "whb_nccl_unique_id": ([ctypes.c_void_p], c_int),
        "whb_nccl_init": ([vp, c_int, c_int, ctypes.c_void_p], c_int),
        "whb_nccl_exchange": ([vp, c_int, ctypes.POINTER(c_u64), ctypes.POINTER(c_u64), ctypes.POINTER(c_i64),
                               ctypes.POINTER(c_int)], c_int),
        "whb_nccl_allreduce_sum": ([vp, dp], c_int),
        "whb_iterate_host": ([vp, dp, dp, dp], c_int),
        "whb_solve_host": ([vp, dp, c_i64, c_i64, dp, c_i64, c_i64, c_int, c_int, dp], c_int),
        "whb_vec_reserve": ([vp, c_int, ctypes.POINTER(c_int)], c_int),
        "whb_vec_upload": ([vp, c_int, dp], c_int),
        "whb_vec_download": ([vp, c_int, dp], c_int),
        "whb_vec_dot": ([vp, c_int, c_int, dp], c_int),
        "whb_vec_axpy": ([vp, c_double, c_int, c_int], c_int),
        "whb_vec_scale_into": ([vp, c_double, c_int, c_int], c_int),
        "whb_vec_div_into": ([vp, c_int, c_double, c_int], c_int),
        "whb_vec_lincomb": ([vp, c_int, c_int, c_int, dp], c_int),
        "whb_vec_sub_into": ([vp, c_int, c_int, c_int], c_int),
        "whb_vec_copy": ([vp, c_int, c_int], c_int),
        "whb_matvec": ([vp, c_int, c_int], c_int),
        "whb_solve_begin": ([vp, c_int, c_int], c_int),
        "whb_step": ([vp, c_int, c_int], c_int),
        "whb_solve_end": ([vp, dp], c_int),
        "whb_level_plane_ptr": ([vp, c_int, c_i64, ctypes.POINTER(c_u64), ip64], c_int),
        "whb_stream_ptr": ([vp, ctypes.POINTER(c_u64)], c_int),
        "whb_synchronize": ([vp], c_int),
        "whb_copy_plane": ([vp, c_int, c_i64, vp, c_int, c_i64], c_int),
        "whb_launch_count": ([vp, ip64], c_int),
        "whb_set_timing": ([vp, c_int], c_int),
        "whb_last_timing": ([vp, dp, ip64, dp], c_int),
        "whb_host_alloc": ([ctypes.POINTER(vp), c_i64], c_int),
        "whb_host_free": ([vp], c_int),
        "whb_geometry": ([vp, ip64, ip64, ip64], c_int),
        "whb_set_l2_flush": ([vp, c_i64], c_int),
        "whb_apply_operator": ([vp, c_int, c_int], c_int),
        "whb_plan": ([vp, ctypes.POINTER(c_int), ctypes.POINTER(c_int)], c_int),
        "whb_set_operator_general": ([vp, c_int, ctypes.POINTER(c_int), dp, c_double], c_int),
        "whb_pair": ([vp, c_int, c_int], c_int),
        "whb_triple": ([vp, c_int, c_int], c_int),
        "whb_ghost_planes": ([vp, ctypes.POINTER(c_int)], c_int),
        "whb_field_plane_ptr": ([vp, c_int, c_int, c_i64, ctypes.POINTER(c_u64), ip64], c_int),
        "whb_copy_device": ([vp, c_u64, vp, c_u64, c_i64], c_int),
        "whb_imp_apply": ([vp, c_int, c_int, c_double, c_int], c_int),
        "whb_imp_rhs": ([vp, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_double, c_double, c_double,
                         c_double], c_int),
        "whb_vec_xpay": ([vp, c_int, c_double, c_int], c_int),
        "whb_mg_setup": ([vp, c_int, ip64, dp, dp, dp, c_int, c_int], c_int),
        "whb_mg_vcycle": ([vp, c_int, c_int], c_int),
        "whb_tri_setup": ([vp, c_int, dp, dp, dp], c_int),
        "whb_tri_solve": ([vp, c_int, c_int], c_int),
        "whb_cg_begin": ([vp, c_int, c_int, c_int, c_int, dp], c_int),
        "whb_vec_mgs": ([vp, c_int, c_int, c_int, c_int, dp], c_int),
        "whb_cg_iterate": ([vp, c_int, c_int, c_int, c_int, c_int, c_int, c_double, c_int, dp, dp], c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(rc: int, what: str = ""):
    if rc == 0:
        return
    msg = load().whb_last_error().decode(errors="replace")
    if rc == E_ARG:
        raise ValueError(f"{what}: {msg}")
    if rc == E_NOMEM:
        raise MemoryError(f"{what}: {msg}")
    raise NativeError(f"{what} failed ({rc}): {msg}")


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = load().whb_device_count(ctypes.byref(n))
    return n.value if rc == 0 else 0


class PinnedBuffer:
    """Page-locked host float64 array (full-rate H2D/D2H)."""

    def __init__(self, shape):
        self.shape = tuple(int(s) for s in shape)
        nbytes = int(np.prod(self.shape)) * 8
        p = ctypes.c_void_p()
        check(load().whb_host_alloc(ctypes.byref(p), nbytes), "whb_host_alloc")
        self._ptr = p
        buf = (ctypes.c_double * max(1, int(np.prod(self.shape)))).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=np.float64, count=int(np.prod(self.shape))).reshape(self.shape)

    def free(self):
        if self._ptr is not None and self._ptr.value:
            load().whb_host_free(self._ptr)
            self._ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class PinnedPool:
    """Recycled page-locked float64 arrays by shape.  An array handed out returns its buffer to the
    pool when the last reference to it (or to any view of it) is gone, so a loop that keeps
    replacing one field by a new one cycles between two pinned buffers instead of paying
    cudaHostAlloc (seconds at 8.6 GB) or pageable transfers (staged by the driver) per call."""

    def __init__(self, keep_per_shape: int = 2, limit_bytes: int = 40 << 30):
        self.keep = keep_per_shape
        self.limit = limit_bytes  # page-locked bytes handed out + pooled (beyond: MemoryError)
        self.free = {}
        self.held = 0

    def empty(self, shape) -> np.ndarray:
        import weakref

        key = tuple(int(x) for x in shape)
        stack = self.free.setdefault(key, [])
        if stack:
            buf = stack.pop()
        else:
            nbytes = int(np.prod(key)) * 8
            if self.held + nbytes > self.limit:
                raise MemoryError("page-locked pool limit reached")
            buf = PinnedBuffer(key)
            self.held += nbytes
        arr = buf.array.view()
        weakref.finalize(arr, self._release, key, buf)
        return arr

    def _release(self, key, buf):
        stack = self.free.setdefault(key, [])
        if len(stack) < self.keep:
            stack.append(buf)
        else:
            self.held -= int(np.prod(key)) * 8
            buf.free()


_pinned_pool = None


def pinned_pool() -> PinnedPool:
    global _pinned_pool
    if _pinned_pool is None:
        _pinned_pool = PinnedPool()
    return _pinned_pool


class Context:
    """Owns one whb_ctx: device buffers for `nbatch` problems on one grid (slab)."""

    def __init__(self, shape, device=0, plane_range=None, nbatch=1, shared_forcing=False):
        L = load()
        self.shape = tuple(int(n) for n in shape)
        self.ndim = len(self.shape)
        if plane_range is None:
            plane_range = (0, self.shape[0] if self.ndim > 1 else 1)
        self.plane_range = (int(plane_range[0]), int(plane_range[1]))
        self.nbatch = int(nbatch)
        self.device = int(device)
        h = ctypes.c_void_p()
        shp = np.array(self.shape, dtype=np.int64)
        check(L.whb_create(ctypes.byref(h), self.device, self.ndim, shp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                           self.plane_range[0], self.plane_range[1], self.nbatch, int(bool(shared_forcing))),
              "whb_create")
        self._hh = h
        # owned part of a field, as host arrays see it
        if self.ndim == 1:
            self.local_shape = self.shape
        else:
            self.local_shape = (self.plane_range[1] - self.plane_range[0],) + self.shape[1:]

    @property
    def _h(self):
        h = getattr(self, "_hh", None)
        if h is None:
            raise RuntimeError("device state released: this context was closed (release_device_cache() or "
                               "close()); create the solver / device problem again")
        return h

    @property
    def handle(self):
        return self._h

    @property
    def closed(self) -> bool:
        return getattr(self, "_hh", None) is None

    def close(self):
        h = getattr(self, "_hh", None)
        if h is not None and h.value:
            load().whb_destroy(h)
        self._hh = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- configuration -------------------------------------------------------------
    def set_operator(self, clo, cmid, c2):
        clo = np.ascontiguousarray(clo, dtype=np.float64)
        cmid = np.ascontiguousarray(cmid, dtype=np.float64)
        check(load().whb_set_operator(self._h, _dp(clo), _dp(cmid), float(c2)), "whb_set_operator")

    def set_operator_general(self, order, periodic, taps, c2):
        per = np.ascontiguousarray(periodic, dtype=np.int32)
        tp = np.ascontiguousarray(taps, dtype=np.float64)
        check(load().whb_set_operator_general(self._h, int(order), per.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                              _dp(tp), float(c2)), "whb_set_operator_general")

    def set_schedule(self, member, sched):
        cos_f = np.ascontiguousarray(sched["cos_f"], dtype=np.float64)
        acc_c = np.ascontiguousarray(sched["acc_c"], dtype=np.float64)
        check(load().whb_set_schedule(self._h, int(member), int(sched["n_total"]), float(sched["half_dt2"]),
                                      float(sched["dt2"]), _dp(cos_f), _dp(acc_c), float(sched["out_scale"])),
              "whb_set_schedule")

    # -- fields --------------------------------------------------------------------
    def _host(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        if a.shape != self.local_shape:
            raise ValueError(f"shape {a.shape} does not match owned field shape {self.local_shape}")
        return a

    def upload(self, field, values, member=0):
        a = self._host(values)
        check(load().whb_upload(self._h, int(field), int(member), _dp(a)), "whb_upload")

    def _out(self, out, what):
        """A caller-supplied output buffer must be exactly what the C ABI writes: float64,
        C-contiguous, the owned field shape (else the D2H copy would overrun it)."""
        if out is None:
            return np.empty(self.local_shape)
        if not isinstance(out, np.ndarray) or out.dtype != np.float64 or not out.flags.c_contiguous \
                or not out.flags.writeable or out.shape != self.local_shape:
            raise ValueError(f"{what}: out must be a writeable C-contiguous float64 array of shape "
                             f"{self.local_shape}")
        return out

    def _in(self, a, what):
        """A host input the C ABI reads in place: float64, C-contiguous, the owned field shape."""
        if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous \
                or a.shape != self.local_shape:
            raise ValueError(f"{what}: expected a C-contiguous float64 array of shape {self.local_shape}")
        return a

    def _strides(self, a):
        """(plane, row) element strides of a float64 view whose last axis is contiguous, in the
        context's storage axes (2D (n0, n1) -> planes = rows of axis 0), or None."""
        if not isinstance(a, np.ndarray) or a.dtype != np.float64 or a.shape != self.local_shape:
            return None
        st = [x // 8 for x in a.strides]
        if a.strides[-1] != 8 or any(x % 8 for x in a.strides):
            return None
        if self.ndim == 3:
            return st[0], st[1]
        if self.ndim == 2:
            return st[0], st[0]
        return None

    def upload_view(self, field, values, member=0):
        """upload() of a strided view (e.g. GridField.values) without packing it on the host."""
        st = None if (isinstance(values, np.ndarray) and values.flags.c_contiguous) else self._strides(values)
        if st is None:
            return self.upload(field, values, member)
        check(load().whb_upload_strided(self._h, int(field), int(member), _dp(values), st[0], st[1]),
              "whb_upload_strided")

    def download_into(self, field, out, member=0):
        """download() straight into a strided writeable view (e.g. a new GridField's interior)."""
        st = None if out.flags.c_contiguous else self._strides(out)
        if st is None or not out.flags.writeable:
            return self.download(field, member, out=out)
        check(load().whb_download_strided(self._h, int(field), int(member), _dp(out), st[0], st[1]),
              "whb_download_strided")
        return out

    def download(self, field, member=0, out=None):
        out = self._out(out, "download")
        check(load().whb_download(self._h, int(field), int(member), _dp(out)), "whb_download")
        return out

    def zero(self, field, member=0):
        check(load().whb_zero(self._h, int(field), int(member)), "whb_zero")

    # -- solves --------------------------------------------------------------------
    def filtered_solve(self, out_mode=OUT_PLAIN, zero_forcing=False):
        r = np.zeros(self.nbatch)
        check(load().whb_filtered_solve(self._h, int(out_mode), int(bool(zero_forcing)), _dp(r)),
              "whb_filtered_solve")
        return r

    def fpi(self, iters, tol_sq=-1.0):
        res = np.zeros(max(1, iters) * self.nbatch)
        done = ctypes.c_int(0)
        check(load().whb_fpi(self._h, int(iters), float(tol_sq), _dp(res), ctypes.byref(done)), "whb_fpi")
        return res[: done.value * self.nbatch].reshape(done.value, self.nbatch)

    def fpi_scaled(self, iters, tol, root_n):
        """Up to `iters` passes, stopping on sqrt(r)/root_n <= tol (driver.py:225-230)."""
        res = np.zeros(max(1, iters) * self.nbatch)
        done = ctypes.c_int(0)
        check(load().whb_fpi_scaled(self._h, int(iters), float(tol), float(root_n), _dp(res), ctypes.byref(done)),
              "whb_fpi_scaled")
        return res[: done.value * self.nbatch].reshape(done.value, self.nbatch)

    def iterate_host(self, v_in, v_out):
        v_in = self._in(v_in, "iterate_host v_in")
        v_out = self._out(v_out, "iterate_host v_out")
        r = np.zeros(1)
        check(load().whb_iterate_host(self._h, _dp(v_in), _dp(v_out), _dp(r)), "whb_iterate_host")
        return float(r[0])

    def solve_host(self, v, out, out_mode=OUT_PLAIN, zero_forcing=False):
        """One filtered solve with host fields on both sides (whb_solve_host): ``v`` and ``out``
        are float64 views of the local shape whose last axis is contiguous (e.g. GridField.values
        and a new field's interior).  Returns resid^2 in FPI mode, else 0."""
        sv, so = self._strides(v), self._strides(out)
        if sv is None or so is None or not out.flags.writeable:
            raise ValueError("solve_host: v / out must be float64 views of the local shape with a contiguous "
                             "last axis (out writeable)")
        r = np.zeros(1)
        check(load().whb_solve_host(self._h, _dp(v), sv[0], sv[1], _dp(out), so[0], so[1], int(out_mode),
                                    int(bool(zero_forcing)), _dp(r)), "whb_solve_host")
        return float(r[0])

    # -- vectors -------------------------------------------------------------------
    def vec_reserve(self, count):
        first = ctypes.c_int(0)
        check(load().whb_vec_reserve(self._h, int(count), ctypes.byref(first)), "whb_vec_reserve")
        return list(range(first.value, first.value + count))

    def vec_upload(self, vid, values):
        a = self._host(values)
        check(load().whb_vec_upload(self._h, int(vid), _dp(a)), "whb_vec_upload")

    def vec_download(self, vid, out=None):
        out = self._out(out, "vec_download")
        check(load().whb_vec_download(self._h, int(vid), _dp(out)), "whb_vec_download")
        return out

    def dot(self, x, y) -> float:
        r = ctypes.c_double(0.0)
        check(load().whb_vec_dot(self._h, int(x), int(y), ctypes.byref(r)), "whb_vec_dot")
        return r.value

    def axpy(self, a, x, y):
        check(load().whb_vec_axpy(self._h, float(a), int(x), int(y)), "whb_vec_axpy")

    def scale_into(self, a, x, y):
        check(load().whb_vec_scale_into(self._h, float(a), int(x), int(y)), "whb_vec_scale_into")

    def div_into(self, x, d, y):
        check(load().whb_vec_div_into(self._h, int(x), float(d), int(y)), "whb_vec_div_into")

    def sub_into(self, x, y, z):
        check(load().whb_vec_sub_into(self._h, int(x), int(y), int(z)), "whb_vec_sub_into")

    def copy(self, x, y):
        check(load().whb_vec_copy(self._h, int(x), int(y)), "whb_vec_copy")

    def lincomb(self, y, first, coef):
        coef = np.ascontiguousarray(coef, dtype=np.float64)
        check(load().whb_vec_lincomb(self._h, int(y), int(first), len(coef), _dp(coef)), "whb_vec_lincomb")

    def apply_operator(self, x, y):
        check(load().whb_apply_operator(self._h, int(x), int(y)), "whb_apply_operator")

    def matvec(self, x, y):
        check(load().whb_matvec(self._h, int(x), int(y)), "whb_matvec")

    # -- step-level control (slab decomposition) ------------------------------------
    # -- implicit stepping -------------------------------------
    def imp_apply(self, x, y, s, tmp=-1):
        check(load().whb_imp_apply(self._h, int(x), int(y), float(s), int(tmp)), "whb_imp_apply")

    def imp_rhs(self, w, wp, lap, f, rhs, guess, first, q0, qh, qd, fs):
        check(load().whb_imp_rhs(self._h, int(w), int(wp), int(lap), int(f), int(rhs), int(guess), int(bool(first)),
                                 float(q0), float(qh), float(qd), float(fs)), "whb_imp_rhs")

    def xpay(self, x, a, y):
        check(load().whb_vec_xpay(self._h, int(x), float(a), int(y)), "whb_vec_xpay")

    def mg_setup(self, cells, gamma, diag, coarse_inv, nu1=2, nu2=2):
        cells = np.ascontiguousarray(np.asarray(cells, dtype=np.int64).reshape(-1))
        gamma = np.ascontiguousarray(np.asarray(gamma, dtype=np.float64).reshape(-1))
        diag = np.ascontiguousarray(diag, dtype=np.float64)
        ainv = np.ascontiguousarray(coarse_inv, dtype=np.float64)
        check(load().whb_mg_setup(self._h, len(diag), cells.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _dp(gamma),
                                  _dp(diag), _dp(ainv), int(nu1), int(nu2)), "whb_mg_setup")

    def mg_vcycle(self, b, u):
        check(load().whb_mg_vcycle(self._h, int(b), int(u)), "whb_mg_vcycle")

    def tri_setup(self, sub, dp_, cp):
        sub = np.ascontiguousarray(sub, dtype=np.float64)
        dp_ = np.ascontiguousarray(dp_, dtype=np.float64)
        cp = np.ascontiguousarray(cp, dtype=np.float64)
        check(load().whb_tri_setup(self._h, len(dp_), _dp(sub), _dp(dp_), _dp(cp)), "whb_tri_setup")

    def tri_solve(self, b, x):
        check(load().whb_tri_solve(self._h, int(b), int(x)), "whb_tri_solve")

    def mgs(self, w, q_first, count, q_next=-1):
        """Device MGS (whb_vec_mgs): returns h[0..count] (h[count] = w.w after projection)."""
        h = np.zeros(count + 1)
        check(load().whb_vec_mgs(self._h, int(w), int(q_first), int(count), int(q_next), _dp(h)), "whb_vec_mgs")
        return h

    def cg_begin(self, r, z, p, precond) -> float:
        rr = ctypes.c_double(0.0)
        check(load().whb_cg_begin(self._h, int(r), int(z), int(p), int(precond), ctypes.byref(rr)), "whb_cg_begin")
        return rr.value

    def cg_iterate(self, x, r, z, p, ap, tmp, s, precond):
        pap = ctypes.c_double(0.0)
        rr = ctypes.c_double(0.0)
        check(load().whb_cg_iterate(self._h, int(x), int(r), int(z), int(p), int(ap), int(tmp), float(s), int(precond),
                                    ctypes.byref(pap), ctypes.byref(rr)), "whb_cg_iterate")
        return pap.value, rr.value

    def solve_begin(self, out_mode, zero_forcing=False):
        check(load().whb_solve_begin(self._h, int(out_mode), int(bool(zero_forcing))), "whb_solve_begin")

    def step(self, s, region=0):
        check(load().whb_step(self._h, int(s), int(region)), "whb_step")

    def pair(self, s, region=0):
        check(load().whb_pair(self._h, int(s), int(region)), "whb_pair")

    def triple(self, s, region=0):
        check(load().whb_triple(self._h, int(s), int(region)), "whb_triple")

    def ghost_planes(self) -> int:
        g = ctypes.c_int(0)
        check(load().whb_ghost_planes(self._h, ctypes.byref(g)), "whb_ghost_planes")
        return g.value

    def field_plane_ptr(self, field, plane, member=0):
        p = ctypes.c_uint64(0)
        n = ctypes.c_int64(0)
        check(load().whb_field_plane_ptr(self._h, int(field), int(member), int(plane), ctypes.byref(p),
                                         ctypes.byref(n)), "whb_field_plane_ptr")
        return p.value, n.value

    def copy_device_to(self, src_ptr: int, dst: "Context", dst_ptr: int, nbytes: int):
        check(load().whb_copy_device(self._h, int(src_ptr), dst._h, int(dst_ptr), int(nbytes)), "whb_copy_device")

    def solve_end(self):
        r = ctypes.c_double(0.0)
        check(load().whb_solve_end(self._h, ctypes.byref(r)), "whb_solve_end")
        return r.value

    def level_plane_ptr(self, level, plane):
        p = ctypes.c_uint64(0)
        n = ctypes.c_int64(0)
        check(load().whb_level_plane_ptr(self._h, int(level), int(plane), ctypes.byref(p), ctypes.byref(n)),
              "whb_level_plane_ptr")
        return p.value, n.value

    # -- peer-memory halo exchange (slab.PeerHalo) ------------------------------------------
    def ipc_handle(self, dev_ptr: int):
        """(64-byte IPC handle of the allocation holding dev_ptr, byte offset of dev_ptr in it)"""
        buf = ctypes.create_string_buffer(64)
        off = ctypes.c_int64(0)
        check(load().whb_ipc_handle(self._h, int(dev_ptr), buf, ctypes.byref(off)), "whb_ipc_handle")
        return buf.raw, off.value

    def ipc_open(self, handle: bytes) -> int:
        p = ctypes.c_uint64(0)
        check(load().whb_ipc_open(self._h, ctypes.create_string_buffer(bytes(handle), 64), ctypes.byref(p)),
              "whb_ipc_open")
        return p.value

    def ipc_close(self, base: int):
        check(load().whb_ipc_close(self._h, int(base)), "whb_ipc_close")

    def flags_alloc(self, count: int) -> int:
        p = ctypes.c_uint64(0)
        check(load().whb_flags_alloc(self._h, int(count), ctypes.byref(p)), "whb_flags_alloc")
        return p.value

    def flags_free(self, ptr: int):
        check(load().whb_flags_free(self._h, int(ptr)), "whb_flags_free")

    def capture_begin(self):
        check(load().whb_capture_begin(self._h), "whb_capture_begin")

    def capture_end(self) -> int:
        g = ctypes.c_int(-1)
        check(load().whb_capture_end(self._h, ctypes.byref(g)), "whb_capture_end")
        return g.value

    def graph_launch(self, graph_id: int):
        check(load().whb_graph_launch(self._h, int(graph_id)), "whb_graph_launch")

    def resid_read(self) -> float:
        r = ctypes.c_double(0.0)
        check(load().whb_resid_read(self._h, ctypes.byref(r)), "whb_resid_read")
        return r.value

    def copy_async(self, src_ptr: int, dst_ptr: int, nbytes: int):
        check(load().whb_copy_async(self._h, int(src_ptr), int(dst_ptr), int(nbytes)), "whb_copy_async")

    def stream_write_u32(self, ptr: int, value: int):
        check(load().whb_stream_write_u32(self._h, int(ptr), int(value) & 0xFFFFFFFF), "whb_stream_write_u32")

    def stream_wait_u32(self, ptr: int, value: int):
        check(load().whb_stream_wait_u32(self._h, int(ptr), int(value) & 0xFFFFFFFF), "whb_stream_wait_u32")

    # -- halo exchange stream and the NCCL path ----------------------------------------
    def comm_begin(self):
        check(load().whb_comm_begin(self._h), "whb_comm_begin")

    def comm_end(self):
        check(load().whb_comm_end(self._h), "whb_comm_end")

    def comm_join(self):
        check(load().whb_comm_join(self._h), "whb_comm_join")

    def nccl_init(self, nranks: int, rank: int, uid: bytes):
        _load_torch_nccl()
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        check(load().whb_nccl_init(self._h, int(nranks), int(rank), buf), "whb_nccl_init")

    def nccl_exchange(self, sends, recvs, counts, peers):
        n = len(sends)
        arr = lambda t, v: (t * max(1, n))(*[int(x) for x in v])  # noqa: E731
        check(load().whb_nccl_exchange(self._h, n, arr(ctypes.c_uint64, sends), arr(ctypes.c_uint64, recvs),
                                       arr(ctypes.c_int64, counts), arr(ctypes.c_int, peers)), "whb_nccl_exchange")

    def nccl_allreduce_sum(self, x: float) -> float:
        v = np.array([float(x)])
        check(load().whb_nccl_allreduce_sum(self._h, _dp(v)), "whb_nccl_allreduce_sum")
        return float(v[0])


    def stream_ptr(self) -> int:
        p = ctypes.c_uint64(0)
        check(load().whb_stream_ptr(self._h, ctypes.byref(p)), "whb_stream_ptr")
        return p.value

    def synchronize(self):
        check(load().whb_synchronize(self._h), "whb_synchronize")

    def copy_plane_to(self, src_level, src_plane, dst: "Context", dst_level, dst_plane):
        check(load().whb_copy_plane(self._h, int(src_level), int(src_plane), dst._h, int(dst_level),
                                    int(dst_plane)), "whb_copy_plane")

    # -- introspection -------------------------------------------------------------
    def launch_count(self) -> int:
        n = ctypes.c_int64(0)
        check(load().whb_launch_count(self._h, ctypes.byref(n)), "whb_launch_count")
        return n.value

    def set_timing(self, on=True):
        check(load().whb_set_timing(self._h, int(bool(on))), "whb_set_timing")

    def last_timing(self):
        a = ctypes.c_double(0.0)
        n = ctypes.c_int64(0)
        b = ctypes.c_double(0.0)
        check(load().whb_last_timing(self._h, ctypes.byref(a), ctypes.byref(n), ctypes.byref(b)),
              "whb_last_timing")
        return a.value, n.value, b.value

    def set_l2_flush(self, nbytes: int):
        check(load().whb_set_l2_flush(self._h, int(nbytes)), "whb_set_l2_flush")

    def plan(self):
        """(kernel, steps_per_pass): kernel 0 simple, 1 bulk rows, 2 TMA tensor boxes."""
        k = ctypes.c_int(0)
        sp = ctypes.c_int(0)
        check(load().whb_plan(self._h, ctypes.byref(k), ctypes.byref(sp)), "whb_plan")
        return k.value, sp.value

    def geometry(self):
        s = np.zeros(3, dtype=np.int64)
        p = ctypes.c_int64(0)
        n = ctypes.c_int64(0)
        check(load().whb_geometry(self._h, s.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ctypes.byref(p),
                                  ctypes.byref(n)), "whb_geometry")
        return tuple(int(x) for x in s), p.value, n.value


def _load_torch_nccl():
    """whb_nccl_* dlopen libnccl.so.2 and reuse a copy the process already loaded: load torch's
    (libtorch_cuda links it) first, so torch and the C ABI share one NCCL -- a system libnccl
    loaded first would shadow torch's newer one (its symbols then fail to resolve)."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    _load_torch_nccl()
    buf = ctypes.create_string_buffer(128)
    check(load().whb_nccl_unique_id(buf), "whb_nccl_unique_id")
    return buf.raw
