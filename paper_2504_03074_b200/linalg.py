"""Restarted GMRES over device-resident vectors — mirror of gmres_solve
(waveholtz/linalg.py:102-183).

Control flow, stopping rules and the residual history follow the reference
line by line; the vector work (mat-vec, modified Gram-Schmidt dot/axpy, norm,
normalisation, solution update) runs on the GPU through the C ABI, and only
the (m+1) x m Hessenberg / Givens scalars live on the host, exactly as in the
reference.  The MGS axpy ``w -= H[j,k]*Q[:,j]`` and the normalisation
``w / h`` are bitwise identical to numpy; dots, norms and the ``Q @ y``
update are deterministic fixed-order reductions (not BLAS-ordered), so
Krylov iterates agree with the reference to rounding.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

__all__ = ["SolveReport", "device_gmres", "gmres_solve"]


@dataclass
class SolveReport:
    """linalg.py:56-66."""

    iterations: int
    relative_residual: float
    converged: bool
    work_units: int = 0
    residual_history: list = field(default_factory=list)
    message: str = ""


def device_gmres(ctx, matvec, b_id: int, x_id: int, tol=1e-10, restart=30, maxit=500, atol=0.0,
                 callback=None, work_ids=None):
    """GMRES on device vectors of ``ctx`` (a ``_native.Context``).

    matvec(src_id, dst_id) writes A*src into dst.  ``x_id`` receives the
    solution (x0 = 0).  ``work_ids`` = [r, Q_0..Q_m] device vector ids
    (reserved here when not given).  Returns a SolveReport.
    """
    report = SolveReport(0, 0.0, True, 0)
    bnorm = math.sqrt(ctx.dot(b_id, b_id))
    target = max(tol * bnorm, atol)
    m_max = max(1, min(restart, maxit))
    if work_ids is None:
        work_ids = ctx.vec_reserve(m_max + 2)
    r_id, q_ids = work_ids[0], work_ids[1:]
    contiguous_basis = all(q_ids[i] == q_ids[0] + i for i in range(len(q_ids)))
    ctx.scale_into(0.0, b_id, x_id)  # x = 0 (b has no NaN/inf)
    if bnorm == 0.0:
        return report

    def mv(src, dst):
        report.work_units += 1
        matvec(src, dst)

    total = 0
    rnorm = bnorm
    while True:
        if total > 0:
            mv(x_id, r_id)
            ctx.sub_into(b_id, r_id, r_id)  # r = b - A x
        else:
            ctx.copy(b_id, r_id)
        rnorm = math.sqrt(ctx.dot(r_id, r_id))
        if total == 0:
            report.residual_history.append(rnorm)
        if rnorm <= target or total >= maxit:
            break
        m = min(restart, maxit - total)
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = rnorm
        ctx.div_into(r_id, rnorm, q_ids[0])  # Q[:,0] = r / rnorm
        k_used = 0
        for k in range(m):
            w = r_id  # workspace reused for w = A Q_k
            mv(q_ids[k], w)
            if contiguous_basis and hasattr(ctx, "mgs"):
                # the whole MGS column on the device, one host round trip (same values as below)
                h = ctx.mgs(w, q_ids[0], k + 1, q_ids[k + 1])
                H[:k + 1, k] = h[:k + 1]
                h_next = math.sqrt(h[k + 1])
            else:
                for j in range(k + 1):
                    H[j, k] = ctx.dot(q_ids[j], w)
                    ctx.axpy(-H[j, k], q_ids[j], w)  # w -= H[j,k]*Q[:,j]
                h_next = math.sqrt(ctx.dot(w, w))
                if h_next > 0:
                    ctx.div_into(w, h_next, q_ids[k + 1])
            H[k + 1, k] = h_next
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
            report.residual_history.append(abs(g[k + 1]))
            if callback is not None:
                callback(abs(g[k + 1]))
            if abs(g[k + 1]) <= target or h_next == 0.0:
                break
        if k_used > 0:
            y = scipy.linalg.solve_triangular(H[:k_used, :k_used], g[:k_used])
            if contiguous_basis:
                ctx.lincomb(x_id, q_ids[0], y)  # x = x + Q[:, :k] @ y (one fused pass)
            else:  # basis ids not consecutive (e.g. caller-provided work_ids): one axpy per vector
                for j in range(k_used):
                    ctx.axpy(float(y[j]), q_ids[j], x_id)
        else:
            break
    report.iterations = total
    report.relative_residual = rnorm / bnorm if bnorm > 0 else rnorm
    report.converged = rnorm <= target
    if not report.converged:
        report.message = f"stagnated after {total} iterations"
    return report


def _host_operator(A):
    if isinstance(A, np.ndarray):
        return lambda x: A @ x
    if hasattr(A, "matvec") and callable(A.matvec):
        return A.matvec
    if callable(A):
        return A
    raise TypeError(f"cannot interpret {type(A)} as a linear operator")


def gmres_solve(A, b, tol=1e-10, restart=30, maxit=500, x0=None, atol=0.0, callback=None):
    """Restarted GMRES with modified Gram-Schmidt Arnoldi and Givens rotations for HOST
    operands (linalg.py:102-183): stops when ||b - A x||_2 <= max(tol*||b||_2, atol); the
    residual history holds the absolute 2-norm after every inner iteration.

    The Krylov basis, the MGS dot/axpy sequence and the solution update run on device vectors
    (device_gmres; the vector is held in the interior of a 1D device field of n + 2 points,
    whose two Dirichlet end points stay 0); ``A`` -- a matrix or a callable on arrays of b's
    shape -- is applied on the host, its operand and result copied per mat-vec.  A nonzero x0
    solves for the correction e = x - x0 from r0 = b - A x0: the same Krylov spaces, iterations
    and residual history as restarting from x0."""
    from . import _native

    op = _host_operator(A)
    b = np.asarray(b, dtype=float)
    shape = b.shape
    n = b.size
    bnorm = float(np.linalg.norm(b.ravel()))
    if bnorm == 0.0 and x0 is None:
        return np.zeros(shape), SolveReport(0, 0.0, True, 0)
    x0v = None if x0 is None else np.array(x0, dtype=float).reshape(shape)
    r0 = b if x0v is None else b - np.asarray(op(x0v), dtype=float).reshape(shape)
    target = max(tol * bnorm, atol)
    ctx = _native.Context((n + 2,))
    try:
        b_id, x_id = ctx.vec_reserve(2)
        pad = np.zeros(n + 2)

        def up(vid, vec):
            pad[1:-1] = np.asarray(vec, dtype=float).ravel()
            ctx.vec_upload(vid, pad)

        def matvec(src, dst):
            v = ctx.vec_download(src)[1:-1].reshape(shape)
            up(dst, np.asarray(op(v), dtype=float))

        up(b_id, r0)
        rep = device_gmres(ctx, matvec, b_id, x_id, tol=0.0, restart=restart, maxit=maxit, atol=target,
                           callback=callback)
        x = ctx.vec_download(x_id)[1:-1].reshape(shape)
    finally:
        ctx.close()
    if x0v is not None:
        x = x0v + x
        r0n = float(np.linalg.norm(r0.ravel()))
        rep.work_units += 1
        rep.relative_residual = rep.relative_residual * r0n / bnorm if bnorm > 0 else rep.relative_residual * r0n
    return x, rep
