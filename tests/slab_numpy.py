"""TEST INFRASTRUCTURE — a numpy stand-in for slab.DeviceShard (and the vector half of the
whb context) with the device's plane layout and region semantics, in reference arithmetic
order.  Used by tests/test_slab_gloo.py and by bench.py --emulate-cpu (the CPU test of the
multi-rank launcher); never by the product path."""

import contextlib

import numpy as np

from paper_2504_03074_b200 import _native
from paper_2504_03074_b200.grid import operator_coefficients


class NumpyShard:
    """Test double with DeviceShard's interface: the same plane layout (G = 3
    ghost planes per side, time level L in buffer L mod 6) and the same
    one-/two-/three-step region semantics as the device contexts
    (include/whb200.h whb_step / whb_pair / whb_triple); arithmetic in
    reference order (the restatement of oracle/waveholtz_oracle.py, per plane)."""

    gh = 3

    def __init__(self, grid, plane_range, c=1.0, steps_per_pass=2):
        self.grid = grid
        self.plane_range = tuple(plane_range)
        self.nloc = plane_range[1] - plane_range[0]
        self.steps_per_pass = steps_per_pass
        self.clo, self.cmid, self.c2 = operator_coefficients(grid, 2, c)
        shp = (self.nloc + 2 * self.gh,) + tuple(grid.shape[1:])
        self.buf = {k: np.zeros(shp) for k in ("v", "f", "acc", "out", 0, 1, 2, 3, 4, 5)}
        self.ctx = NumpyVecs(self)
        self.zf = False
        self.device = 0
        n0, g, p0 = grid.shape[0], self.gh, plane_range[0]
        g_lo, g_hi = max(plane_range[0], 1), min(plane_range[1], n0 - 1)
        self.lo, self.hi = g_lo - p0 + g, max(g_hi - p0 + g, g_lo - p0 + g)
        # global-interior planes in local indices (W^{s+1} of ghost planes is computed there)
        self.i_lo, self.i_hi = max(0, 1 - p0 + g), min(shp[0], n0 - 1 - p0 + g)

    def set_schedule(self, sched):
        self.sc = sched
        self.n_total = sched["n_total"]

    def _field(self, field):
        return {_native.V: "v", _native.F: "f", _native.ACC: "acc", _native.OUT: "out"}[field]

    def upload(self, field, vals):
        a = np.array(vals, dtype=float)
        for ax in range(1, a.ndim):
            sl = [slice(None)] * a.ndim
            for e in (0, -1):
                sl[ax] = e
                a[tuple(sl)] = 0.0
        if self.plane_range[0] == 0:
            a[0] = 0.0
        if self.plane_range[1] == self.grid.shape[0]:
            a[-1] = 0.0
        self.buf[self._field(field)][self.gh:self.gh + self.nloc] = a

    def download(self, field):
        return np.array(self.buf[self._field(field)][self.gh:self.gh + self.nloc])

    def zero(self, field):
        self.buf[self._field(field)][...] = 0.0

    def level(self, L):
        return self.buf["v"] if L == 0 else self.buf[L % 6]

    def solve_begin(self, out_mode, zero_forcing=False):
        self.mode = out_mode
        self.zf = bool(zero_forcing) or out_mode == _native.OUT_AV
        self.rs = 0.0

    def _lap(self, w, i):
        lap = 0.0
        lap = lap + self.clo[0] * w[i - 1][..., 1:-1]
        lap = lap + self.cmid[0] * w[i][..., 1:-1]
        lap = lap + self.clo[0] * w[i + 1][..., 1:-1]
        if w.ndim == 3:
            lap = lap[1:-1]
            lap = lap + self.clo[1] * w[i][:-2, 1:-1]
            lap = lap + self.cmid[1] * w[i][1:-1, 1:-1]
            lap = lap + self.clo[1] * w[i][2:, 1:-1]
            c = w[i][1:-1]
        else:
            c = w[i]
        lap = lap + self.clo[-1] * c[..., :-2]
        lap = lap + self.cmid[-1] * c[..., 1:-1]
        lap = lap + self.clo[-1] * c[..., 2:]
        if self.c2 != 1.0:
            lap = lap * self.c2
        return lap

    def _inner(self):
        return (slice(1, -1),) * (self.buf["v"].ndim - 1)

    def _advance(self, s, w, wp, i):
        """interior of W^{s+1} at plane i from W^s (w) and W^{s-1} (wp)"""
        sc, inner = self.sc, self._inner()
        lap = self._lap(w, i)
        f = self.buf["f"][i][inner] * 0.0 if self.zf else self.buf["f"][i][inner]
        wc = w[i][inner]
        if s == 0:
            return wc + sc["half_dt2"] * (lap - f)
        return 2.0 * wc - wp[i][inner] + sc["dt2"] * (lap - f * sc["cos_f"][s])

    def _finish(self, s, i, w, new):
        """filter update of step s at plane i (W^s = w, W^{s+1} interior = new); returns
        True when the value must also be stored as W^{s+1}"""
        sc, inner = self.sc, self._inner()
        acc = self.buf["acc"][i]
        if s == 0:
            acc[inner] = sc["acc_c"][0] * w[i][inner]
        acc[inner] = acc[inner] + sc["acc_c"][s + 1] * new
        if s == self.n_total - 1:
            out = sc["out_scale"] * acc[inner]
            if self.mode == _native.OUT_FPI:
                d = out - self.buf["v"][i][inner]
                self.rs += float(np.sum(d * d))
                self.buf["v"][i][inner] = out
            elif self.mode == _native.OUT_AV:
                self.buf["out"][i][inner] = self.buf["v"][i][inner] - out
            else:
                self.buf["out"][i][inner] = out
            return False
        return True

    def step(self, s, region):
        lo, hi = self.lo, self.hi
        planes = {0: range(lo, hi), 1: sorted({lo, hi - 1}) if hi > lo else [], 2: range(lo + 1, hi - 1)}[region]
        w, wp, wn = self.level(s), self.level(s - 1), self.level(s + 1)
        inner = self._inner()
        for i in planes:
            new = self._advance(s, w, wp, i)
            if self._finish(s, i, w, new):
                wn[i][inner] = new

    def _pair_range(self, s, a, b):
        """steps s, s+1 on update planes [a, b): W^{s+1} on [a-1, b] (zero outside the global
        interior, kept aside), then W^{s+2} on [a, b) — what one chunk of the device pass does"""
        w, wp = self.level(s), self.level(s - 1)
        inner = self._inner()
        w1 = np.zeros_like(w)
        for i in range(a - 1, b + 1):
            if self.i_lo <= i < self.i_hi:
                w1[i][inner] = self._advance(s, w, wp, i)
        for i in range(a, b):
            self._finish(s, i, w, w1[i][inner])
            self.level(s + 1)[i][inner] = w1[i][inner]
            new = self._advance(s + 1, w1, w, i)
            if self._finish(s + 1, i, w1, new):
                self.level(s + 2)[i][inner] = new

    def pair(self, s, region):
        lo, hi = self.lo, self.hi
        if region == 0:
            self._pair_range(s, lo, hi)
        elif region == 1:
            if hi - lo <= 4:
                self._pair_range(s, lo, hi)
            else:
                self._pair_range(s, lo, lo + 2)
                self._pair_range(s, hi - 2, hi)
        elif hi - lo > 4:
            self._pair_range(s, lo + 2, hi - 2)

    def _triple_range(self, s, a, b):
        """steps s, s+1, s+2 on update planes [a, b): W^{s+1} on [a-2, b+2) and W^{s+2} on
        [a-1, b+1) (zero outside the global interior, kept aside), then W^{s+3} on [a, b); W^{s+2}
        and W^{s+3} of [a, b) are stored (what the next pass reads) — one chunk of the device pass"""
        w, wp = self.level(s), self.level(s - 1)
        inner = self._inner()
        w1, w2 = np.zeros_like(w), np.zeros_like(w)
        for i in range(a - 2, b + 2):
            if self.i_lo <= i < self.i_hi:
                w1[i][inner] = self._advance(s, w, wp, i)
        for i in range(a - 1, b + 1):
            if self.i_lo <= i < self.i_hi:
                w2[i][inner] = self._advance(s + 1, w1, w, i)
        for i in range(a, b):
            self._finish(s, i, w, w1[i][inner])
            self._finish(s + 1, i, w1, w2[i][inner])
            self.level(s + 2)[i][inner] = w2[i][inner]
            new = self._advance(s + 2, w2, w1, i)
            if self._finish(s + 2, i, w2, new):
                self.level(s + 3)[i][inner] = new

    def triple(self, s, region):
        lo, hi = self.lo, self.hi
        if region == 0:
            self._triple_range(s, lo, hi)
        elif region == 1:
            if hi - lo <= 6:
                self._triple_range(s, lo, hi)
            else:
                self._triple_range(s, lo, lo + 3)
                self._triple_range(s, hi - 3, hi)
        elif hi - lo > 6:
            self._triple_range(s, lo + 3, hi - 3)

    def solve_end(self):
        return self.rs

    def planes(self, item, first, count):
        import torch

        kind, ident = item
        arr = self.level(ident) if kind == "level" else self.buf[self._field(ident)]
        return torch.from_numpy(arr[first:first + count].reshape(-1))

    def stream(self):
        return contextlib.nullcontext()


class NumpyVecs:
    """The vector half of the whb context interface (ids 0..7 alias the shard's fields,
    ids >= 8 are extra vectors) over a NumpyShard's owned planes."""

    def __init__(self, shard):
        self.sh = shard
        self.extra = []

    def _a(self, vid):
        if vid >= 8:
            return self.extra[vid - 8]
        return self.sh.buf[self.sh._field(vid)]

    def _own(self, vid):
        g = self.sh.gh
        return self._a(vid)[g:g + self.sh.nloc]

    def vec_reserve(self, count):
        first = 8 + len(self.extra)
        self.extra += [np.zeros_like(self.sh.buf["v"]) for _ in range(count)]
        return list(range(first, first + count))

    def vec_download(self, vid):
        return np.array(self._own(vid))

    def dot(self, x, y):
        return float(np.sum(self._own(x) * self._own(y)))

    def axpy(self, a, x, y):
        self._own(y)[...] = self._own(y) - (-a) * self._own(x)

    def scale_into(self, a, x, y):
        self._own(y)[...] = self._own(x) * a

    def div_into(self, x, d, y):
        self._own(y)[...] = self._own(x) / d

    def sub_into(self, x, y, z):
        self._own(z)[...] = self._own(x) - self._own(y)

    def copy(self, x, y):
        self._a(y)[...] = self._a(x)

    def lincomb(self, y, first, coef):
        acc = self._own(y)
        for j, c in enumerate(coef):
            acc = acc + c * self._own(first + j)
        self._own(y)[...] = acc
