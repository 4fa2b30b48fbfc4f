"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference's explicit WaveHoltz path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu baseline /
``--impl reference``) may use this module, and only as the checker or the timed
CPU baseline.  The product package never imports it.

Every function follows the reference's operation order exactly, so its
results are bitwise identical to ``waveholtz`` 0.1.0 (pinned against the
golden fixtures in ``tests/golden`` — see ``tests/test_oracle_golden.py``).
Third-party dependency holding the arithmetic: numpy (reference pins
``numpy>=1.24``, pkg/pyproject.toml:10-13; this image has 2.3.5).  Elementwise
ufuncs are separately rounded IEEE ops, so the order below is all that matters.
"""

from __future__ import annotations

import math

import numpy as np

# timestep.py:43 — Courant numbers of leap-frog with order-p space discretisation
COURANT = {2: 1.0, 4: math.sqrt(3.0) / 2.0}


# ---------------------------------------------------------------------------------
# host scalars


def alpha_d(omega_dt: float) -> float:
    """filters.py:160-166."""
    if not 0.0 < omega_dt < math.pi / 2.0:
        raise ValueError("omega*dt outside (0, pi/2)")
    return math.tan(omega_dt / 2.0) / math.tan(omega_dt)


def correct_explicit(omega: float, spacing, p: int = 2, c: float = 1.0, courant: float | None = None):
    """timestep.py:78-97 -> (N_t, dt, omega_e).  ``courant`` overrides _COURANT[p]."""
    if not omega > 0:
        raise ValueError("omega must be positive")
    inv_sq = sum(1.0 / dx**2 for dx in spacing)
    cfl = COURANT[p] if courant is None else courant
    bound = cfl**2
    dt_max = math.sqrt(bound / (c**2 * inv_sq))
    n_t = max(5, math.ceil(2.0 * math.pi / omega / dt_max))
    while True:
        dt = (2.0 / omega) * math.sin(math.pi / n_t)
        if c**2 * dt**2 * inv_sq < bound:
            break
        n_t += 1
    omega_e = 2.0 * math.pi / (n_t * dt)
    return n_t, dt, omega_e


def step_scalars(n_t: int, dt: float, omega_e: float, periods: int = 1):
    """Per-step scalars exactly as wave_solve_filtered forms them.

    Returns dict(n_total, half_dt2, dt2, cos_f[n_total], acc_c[n_total+1], out_scale).
    cos_f[n] = cos(wt*(n*dt)) for the forcing of step n (timestep.py:139, t = n*dt
    set at timestep.py:144); acc_c[n] = (cos(wt*(n*dt)) - 0.5*alpha)*sigma_n
    (timestep.py:284, 297-298); out_scale = (2/t_bar)*dt (timestep.py:277, 300).
    """
    alpha = alpha_d(omega_e * dt)  # timestep.py:73-75
    n_total = periods * n_t
    cos_f = np.empty(n_total)
    cos_f[0] = 1.0  # unused (first step carries no cos factor, timestep.py:137)
    for n in range(1, n_total):
        cos_f[n] = math.cos(omega_e * (n * dt))
    acc_c = np.empty(n_total + 1)
    acc_c[0] = (math.cos(0.0) - 0.5 * alpha) * 0.5
    for n in range(1, n_total + 1):
        sigma = 0.5 if n == n_total else 1.0
        acc_c[n] = (math.cos(omega_e * (n * dt)) - 0.5 * alpha) * sigma
    t_bar = n_total * dt
    return {
        "n_total": n_total,
        "half_dt2": 0.5 * dt**2,
        "dt2": dt**2,
        "cos_f": cos_f,
        "acc_c": acc_c,
        "out_scale": (2.0 / t_bar) * dt,
        "alpha": alpha,
    }


# ---------------------------------------------------------------------------------
# fields


def coords(shape, bounds, spacing):
    """grid.py:104-112 (meshgrid 'ij')."""
    axes = [lo + dx * np.arange(n) for (lo, _), dx, n in zip(bounds, spacing, shape)]
    return tuple(np.meshgrid(*axes, indexing="ij")) if len(shape) > 1 else (axes[0],)


def zero_boundary(a: np.ndarray) -> np.ndarray:
    """grid.py:237-246 / 395-402 (all-Dirichlet)."""
    for axis in range(a.ndim):
        idx = [slice(None)] * a.ndim
        idx[axis] = 0
        a[tuple(idx)] = 0.0
        idx[axis] = -1
        a[tuple(idx)] = 0.0
    return a


def gaussian(shape, bounds, spacing, a_g, b_g, x0):
    """driver.py:163-179: a_g*exp(-b_g*r2), r2 accumulated axis by axis from 0."""
    cs = coords(shape, bounds, spacing)
    r2 = np.zeros(shape)
    for ax in range(len(shape)):
        r2 = r2 + (cs[ax] - x0[ax]) ** 2
    return zero_boundary(np.array(a_g * np.exp(-b_g * r2)))


def multi_gaussian(shape, bounds, spacing, n_gauss, seed=0):
    """BASELINE forcing recipe."""
    d = len(shape)
    rng = np.random.default_rng(seed)
    amp = rng.uniform(-100.0, 100.0, n_gauss)
    ctr = rng.uniform(0.1, 0.9, (n_gauss, d))
    b = rng.uniform(100.0, 1000.0, n_gauss)
    f = np.zeros(shape)
    for k in range(n_gauss):
        f = f + gaussian(shape, bounds, spacing, amp[k], b[k], ctr[k])
    return zero_boundary(f)


# ---------------------------------------------------------------------------------
# operator + stepping


def laplacian(w: np.ndarray, spacing, c: float = 1.0) -> np.ndarray:
    """grid.py:346-368 + 371-392 (p=2, all Dirichlet): pad with odd reflection,
    out = 0; for axis: for tap k: out += (s_k/dx^2)*buf[shift]; out *= c^2; zero boundary."""
    g = 1
    buf = np.empty(tuple(n + 2 * g for n in w.shape))
    core = tuple(slice(g, g + n) for n in w.shape)
    buf[core] = w
    for axis, n in enumerate(w.shape):
        def ax(idx):
            sl = [slice(g, g + m) for m in w.shape]
            sl[axis] = idx
            return tuple(sl)
        buf[ax(g - 1)] = -buf[ax(g + 1)]
        buf[ax(g + n)] = -buf[ax(g + n - 2)]
    out = np.zeros(w.shape)
    for axis, dx in enumerate(spacing):
        taps = np.array([1.0, -2.0, 1.0]) / dx**2
        for k, ck in enumerate(taps):
            off = k - 1
            sl = list(core)
            sl[axis] = slice(g + off, g + off + w.shape[axis])
            out += ck * buf[tuple(sl)]
    out *= c**2
    return zero_boundary(out)


TAPS = {2: np.array([1.0, -2.0, 1.0]),
        4: np.array([-1.0 / 12.0, 4.0 / 3.0, -5.0 / 2.0, 4.0 / 3.0, -1.0 / 12.0])}


def zero_dirichlet(a: np.ndarray, bcs) -> np.ndarray:
    """grid.py:395-402 for per-axis boundary conditions."""
    for axis, bc in enumerate(bcs):
        if bc == "dirichlet":
            idx = [slice(None)] * a.ndim
            for e in (0, -1):
                idx[axis] = e
                a[tuple(idx)] = 0.0
    return a


def laplacian_general(w: np.ndarray, spacing, bcs, order: int = 2, c: float = 1.0) -> np.ndarray:
    """grid.py:346-392 for order p in {2, 4} and per-axis Dirichlet / periodic boundaries:
    ghosts of width p/2 by odd reflection (Dirichlet) or wrap (periodic), filled axis by
    axis over the core of the other axes; out = 0; per axis, per tap: out += c_k*buf[shift];
    out *= c^2; Dirichlet faces zeroed."""
    g = order // 2
    shape = w.shape
    buf = np.empty(tuple(n + 2 * g for n in shape))
    core = tuple(slice(g, g + n) for n in shape)
    buf[core] = w
    for axis, bc in enumerate(bcs):
        n = shape[axis]

        def ax(idx):
            sl = [slice(g, g + m) for m in shape]
            sl[axis] = idx
            return tuple(sl)

        for k in range(1, g + 1):
            if bc == "dirichlet":
                buf[ax(g - k)] = -buf[ax(g + k)]
                buf[ax(g + n - 1 + k)] = -buf[ax(g + n - 1 - k)]
            else:
                buf[ax(g - k)] = buf[ax(g + n - k)]
                buf[ax(g + n - 1 + k)] = buf[ax(g + k - 1)]
    out = np.zeros(shape)
    for axis, dx in enumerate(spacing):
        taps = TAPS[order] / dx**2
        for k, ck in enumerate(taps):
            off = k - g
            sl = list(core)
            sl[axis] = slice(g + off, g + off + shape[axis])
            out += ck * buf[tuple(sl)]
    out *= c**2
    return zero_dirichlet(out, bcs)


def wave_solve_filtered(v: np.ndarray, f: np.ndarray, spacing, sc: dict, c: float = 1.0, bcs=None,
                        order: int = 2) -> np.ndarray:
    """timestep.py:250-301, explicit branch, with step_explicit (timestep.py:132-145)."""
    n_total = sc["n_total"]
    w = np.array(v, dtype=float)
    w_prev = np.zeros_like(w)
    acc = sc["acc_c"][0] * w
    general = bcs is not None or order != 2
    bcs = bcs or ["dirichlet"] * w.ndim
    for n in range(n_total):
        lap = laplacian_general(w, spacing, bcs, order, c) if general else laplacian(w, spacing, c)
        if n == 0:
            w_next = w + sc["half_dt2"] * (lap - f)
        else:
            force = f * sc["cos_f"][n]
            w_next = 2.0 * w - w_prev + sc["dt2"] * (lap - force)
        w_prev, w = w, w_next
        acc += sc["acc_c"][n + 1] * w
    return zero_dirichlet(sc["out_scale"] * acc, bcs)


def fpi(f: np.ndarray, spacing, sc: dict, iters: int, c: float = 1.0, tol: float = -1.0):
    """driver.py:211-230: v0 = 0, v <- W(v, f), residual ||v_new - v||_2/sqrt(N)."""
    v = np.zeros_like(f)
    res = []
    for _ in range(iters):
        v_new = wave_solve_filtered(v, f, spacing, sc, c)
        diff = np.linalg.norm(v_new - v) / math.sqrt(v.size)
        res.append(diff)
        v = v_new
        if diff <= tol:
            break
    return v, res


def apply_A(x: np.ndarray, spacing, sc: dict, c: float = 1.0, bcs=None, order: int = 2) -> np.ndarray:
    """driver.py:256-262: A x = x - W(x, 0)."""
    return x - wave_solve_filtered(x, np.zeros_like(x), spacing, sc, c, bcs, order)


# ---------------------------------------------------------------------------------
# analytic known-answer tests (independent of any stepping)


def sinc_d(z, T, dt):
    """filters.py:134-157."""
    n_ratio = T / dt
    n = round(n_ratio)
    phi = np.asarray(z, dtype=float) * dt / 2.0
    m = np.round(phi / np.pi)
    d = phi - m * np.pi
    tiny = np.abs(d) < 1e-300
    safe_d = np.where(tiny, 1.0, d)
    val = np.where(tiny, 1.0, np.sin(2.0 * n * safe_d) * np.cos(safe_d) / (2.0 * n * np.sin(safe_d)))
    return val


def beta_d(lam, omega, T, n_t, alpha):
    """filters.py:169-182."""
    dt = T / n_t
    return sinc_d(omega + lam, T, dt) + sinc_d(omega - lam, T, dt) - alpha * sinc_d(lam, T, dt)


def lambda_tilde_explicit(lam_h, dt):
    """filters.py:205-215."""
    return (2.0 / dt) * np.arcsin(np.asarray(lam_h) * dt / 2.0)


def sine_mode(cells, lengths, ks):
    """grid.py:475-496 (Dirichlet sine mode, volume-orthonormal) as a dense array."""
    vals = None
    for n, L, m in zip(cells, lengths, ks):
        j = np.arange(n + 1)
        v = np.sin(m * np.pi * j / n) * np.sqrt(2.0 / L)
        vals = v if vals is None else np.multiply.outer(vals, v)
    return vals


def sine_mode_lambda(cells, spacing, ks, c=1.0):
    """grid.py:417-435: lambda^2 = sum_m (c/dx_m)^2 * 4 sin^2(k_m pi/(2 n_m))."""
    lam2 = 0.0
    for n, dx, m in zip(cells, spacing, ks):
        lam2 += (c / dx) ** 2 * 4.0 * math.sin(m * math.pi / n / 2.0) ** 2
    return math.sqrt(lam2)


def eigen_action_factor(cells, spacing, ks, omega, n_t, dt, omega_e, periods=1, c=1.0):
    """W(phi, 0) = beta_d(lambda_e) phi (test_timestep.py:220-236)."""
    lam = sine_mode_lambda(cells, spacing, ks, c)
    lam_e = float(lambda_tilde_explicit(lam, dt))
    alpha = alpha_d(omega_e * dt)
    T = periods * n_t * dt
    return float(beta_d(lam_e, omega_e, T, periods * n_t, alpha))


# ---------------------------------------------------------------------------------
# GMRES (linalg.py:102-183) on numpy vectors — oracle for the device Krylov path


def gmres(matvec, b, tol=1e-10, restart=30, maxit=500, atol=0.0):
    import scipy.linalg

    shape = b.shape
    bvec = b.ravel()
    n = bvec.size
    bnorm = np.linalg.norm(bvec)
    target = max(tol * bnorm, atol)
    hist = []
    if bnorm == 0.0:
        return np.zeros(shape), hist, 0, True
    x = np.zeros(n)
    total = 0
    while True:
        r = bvec - matvec(x.reshape(shape)).ravel() if total > 0 else bvec.copy()
        rnorm = np.linalg.norm(r)
        if total == 0:
            hist.append(rnorm)
        if rnorm <= target or total >= maxit:
            break
        m = min(restart, maxit - total)
        Q = np.empty((n, m + 1))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = rnorm
        Q[:, 0] = r / rnorm
        k_used = 0
        for k in range(m):
            w = matvec(Q[:, k].reshape(shape)).ravel()
            for j in range(k + 1):
                H[j, k] = np.vdot(Q[:, j], w)
                w -= H[j, k] * Q[:, j]
            h_next = np.linalg.norm(w)
            H[k + 1, k] = h_next
            if h_next > 0:
                Q[:, k + 1] = w / h_next
            for j in range(k):
                t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
                H[j + 1, k] = -sn[j] * H[j, k] + cs[j] * H[j + 1, k]
                H[j, k] = t
            denom = np.hypot(H[k, k], H[k + 1, k])
            if denom == 0.0:
                k_used = k
                break
            cs[k] = H[k, k] / denom
            sn[k] = H[k + 1, k] / denom
            H[k, k] = denom
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            k_used = k + 1
            total += 1
            hist.append(abs(g[k + 1]))
            if abs(g[k + 1]) <= target or h_next == 0.0:
                break
        if k_used > 0:
            y = scipy.linalg.solve_triangular(H[:k_used, :k_used], g[:k_used])
            x = x + Q[:, :k_used] @ y
        else:
            break
    return x.reshape(shape), hist, total, rnorm <= target
