// Implicit trapezoidal stepping: the kernels under
// waveholtz/timestep.py:148-247 and linalg.py:189-370.
//
// Each implicit step solves (I - (dt^2/2) c^2 L_h) W^{n+1} = rhs.  The
// reference solves it with CG (linalg.py:62-99) preconditioned by one
// geometric-multigrid V-cycle (2D, all-Dirichlet: red-black Gauss-Seidel,
// full-weighting restriction, bilinear prolongation, dense coarse solve) or by
// the exact tridiagonal elimination (1D), or directly by that elimination
// (1D, p = 2).  The kernels below are those pieces; the CG loop itself runs on
// the host over device vectors (paper_2504_03074_b200/implicit.py), like the
// reference's.  Elementwise values follow the reference's operation order;
// reductions (CG dots/norms) use the fixed-order device tree, so implicit
// iterates match the reference to the inner-solve tolerance (not bitwise).
//
// Multigrid level arrays are row-major (nx+1) x (ny+1) with a row stride rs:
// level 0 is the context's own 2D field layout (rows = storage planes,
// rs = pitch), coarser levels are compact pitched arrays.
#pragma once

namespace imp {

// y = x - s * (c^2 L_h x); L_h x = 0 at Dirichlet points (timestep.py:225-226 `apply`,
// grid.py:346-368).  Owned planes [lp0, lp1), update planes [up0, up1).
template <bool A0, bool A1>
__global__ void apply_kernel(Geom g, const double *__restrict__ x, double *__restrict__ y, double s, int lp0,
                             int lp1, int up0, int up1) {
    const long long total = (long long)(lp1 - lp0) * g.S0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long pl = t / g.S0;
        const long long r = t - pl * g.S0;
        const int j = (int)(r / g.P);
        const int k = (int)(r - (long long)j * g.P);
        if (k >= g.n2) continue;  // row padding stays 0
        const int plane = lp0 + (int)pl;
        const long long p = (long long)plane * g.S0 + r;
        const double xc = x[p];
        double lap = 0.0;
        const bool in = (k >= 1 && k < g.n2 - 1) && (!A1 || (j >= g.j_lo && j < g.j_hi)) &&
                        (!A0 || (plane >= up0 && plane < up1));
        if (in) {
            if (A0) {
                lap = whb_add(lap, whb_mul(g.clo0, x[p - g.S0]));
                lap = whb_add(lap, whb_mul(g.cmid0, xc));
                lap = whb_add(lap, whb_mul(g.clo0, x[p + g.S0]));
            }
            if (A1) {
                lap = whb_add(lap, whb_mul(g.clo1, x[p - g.P]));
                lap = whb_add(lap, whb_mul(g.cmid1, xc));
                lap = whb_add(lap, whb_mul(g.clo1, x[p + g.P]));
            }
            lap = whb_add(lap, whb_mul(g.clo2, x[p - 1]));
            lap = whb_add(lap, whb_mul(g.cmid2, xc));
            lap = whb_add(lap, whb_mul(g.clo2, x[p + 1]));
            lap = whb_mul(lap, g.c2);  // out *= c**2 (grid.py:366)
        }
        y[p] = whb_sub(xc, whb_mul(s, lap));
    }
}

// y = x - s * t (the general-operator form of apply_kernel: t = c^2 L_h x, 0 at boundaries)
__global__ void sub_scaled_kernel(const double *__restrict__ x, double s, const double *__restrict__ t,
                                  double *__restrict__ y, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = whb_sub(x[i], whb_mul(s, t[i]));
}

// Right-hand side and initial guess of one implicit step (timestep.py:155-164):
//   n = 0: rhs = w - q0*f, guess = w                (q0 = (0.5*dt**2)*cos_fac)
//   n > 0: rhs = ((2w - wp) + qh*lap) - qd*(f*fs), guess = 2w - wp
//          (qh = 0.5*dt**2, qd = dt**2, fs = cos(wt*t)*cos_fac, lap = c^2 L_h wp)
__global__ void rhs_kernel(const double *__restrict__ w, const double *__restrict__ wp,
                           const double *__restrict__ lap, const double *__restrict__ f, double *__restrict__ rhs,
                           double *__restrict__ guess, int first, double q0, double qh, double qd, double fs,
                           long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double wv = w[i];
        if (first) {
            rhs[i] = whb_sub(wv, whb_mul(q0, f[i]));
            guess[i] = wv;
        } else {
            const double t1 = whb_sub(whb_mul(2.0, wv), wp[i]);
            rhs[i] = whb_sub(whb_add(t1, whb_mul(qh, lap[i])), whb_mul(qd, whb_mul(f[i], fs)));
            guess[i] = t1;
        }
    }
}

// y = x + a*y (CG direction update p = z + beta*p, linalg.py:97)
__global__ void xpay_kernel(const double *__restrict__ x, double a, double *y, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = whb_add(x[i], whb_mul(a, y[i]));
}

// ---- 2D multigrid levels (linalg.py:189-283) -------------------------------------------------

struct Lev {
    int nx, ny;      // cells per axis (points nx+1, ny+1)
    long long rs;    // row stride (elements)
    double gx, gy, diag;
};

// r = b - A u (A u = 0 at boundary points) over the whole level (linalg.py:206-217, 333)
__global__ void residual_kernel(Lev L, const double *__restrict__ u, const double *__restrict__ b,
                                double *__restrict__ r) {
    const long long total = (long long)(L.nx + 1) * (L.ny + 1);
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(t / (L.ny + 1));
        const int j = (int)(t - (long long)i * (L.ny + 1));
        const long long p = (long long)i * L.rs + j;
        double au = 0.0;
        if (i >= 1 && i < L.nx && j >= 1 && j < L.ny) {
            au = whb_sub(whb_sub(whb_mul(L.diag, u[p]), whb_mul(L.gx, whb_add(u[p - L.rs], u[p + L.rs]))),
                         whb_mul(L.gy, whb_add(u[p - 1], u[p + 1])));
        }
        r[p] = whb_sub(b[p], au);
    }
}

// one red-black colour: points with (i + j) % 2 == colour (linalg.py:230-238)
__global__ void gs_color_kernel(Lev L, double *__restrict__ u, const double *__restrict__ b, int color) {
    const int half = L.ny / 2 + 1;
    const long long total = (long long)(L.nx - 1) * half;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = 1 + (int)(t / half);
        const int m = (int)(t - (long long)(i - 1) * half);
        const int j = 2 * m + ((i + color) & 1);
        if (j < 1 || j >= L.ny) continue;
        const long long p = (long long)i * L.rs + j;
        const double v = whb_add(whb_add(b[p], whb_mul(L.gx, whb_add(u[p - L.rs], u[p + L.rs]))),
                                 whb_mul(L.gy, whb_add(u[p - 1], u[p + 1])));
        u[p] = __ddiv_rn(v, L.diag);
    }
}

// full-weighting restriction of the fine residual r onto the coarse level (boundary 0)
// (linalg.py:247-257)
__global__ void restrict_kernel(Lev F, const double *__restrict__ r, Lev C, double *__restrict__ rc) {
    const long long total = (long long)(C.nx + 1) * (C.ny + 1);
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int I = (int)(t / (C.ny + 1));
        const int J = (int)(t - (long long)I * (C.ny + 1));
        double v = 0.0;
        if (I >= 1 && I < C.nx && J >= 1 && J < C.ny) {
            const long long p = (long long)(2 * I) * F.rs + 2 * J;
            const long long rs = F.rs;
            const double edges = whb_add(whb_add(whb_add(r[p - rs], r[p + rs]), r[p - 1]), r[p + 1]);
            const double corners = whb_add(whb_add(whb_add(r[p - rs - 1], r[p - rs + 1]), r[p + rs - 1]), r[p + rs + 1]);
            v = __ddiv_rn(whb_add(whb_add(whb_mul(4.0, r[p]), whb_mul(2.0, edges)), corners), 16.0);
        }
        rc[(long long)I * C.rs + J] = v;
    }
}

// u += prolong(ec) (bilinear, linalg.py:259-275, 337)
__global__ void prolong_add_kernel(Lev F, double *__restrict__ u, Lev C, const double *__restrict__ ec) {
    const long long total = (long long)(F.nx + 1) * (F.ny + 1);
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(t / (F.ny + 1));
        const int j = (int)(t - (long long)i * (F.ny + 1));
        const int a = i >> 1, bq = j >> 1;
        const long long q = (long long)a * C.rs + bq;
        double e;
        if (!(i & 1) && !(j & 1)) e = ec[q];
        else if ((i & 1) && !(j & 1)) e = whb_mul(0.5, whb_add(ec[q], ec[q + C.rs]));
        else if (!(i & 1) && (j & 1)) e = whb_mul(0.5, whb_add(ec[q], ec[q + 1]));
        else e = whb_mul(0.25, whb_add(whb_add(whb_add(ec[q], ec[q + C.rs]), ec[q + 1]), ec[q + C.rs + 1]));
        const long long p = (long long)i * F.rs + j;
        u[p] = whb_add(u[p], e);
    }
}

// coarsest level: u = scatter(Ainv @ interior(b)); one warp per interior unknown
// (linalg.py:316-319 uses an LU solve of the same matrix)
__global__ void coarse_solve_kernel(Lev C, const double *__restrict__ ainv, const double *__restrict__ b,
                                    double *__restrict__ u) {
    const int mi = C.ny - 1;
    const int n = (C.nx - 1) * mi;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int k = warp; k < n; k += nw) {
        double s = 0.0;
        for (int l = lane; l < n; l += 32) {
            const int I = 1 + l / mi, J = 1 + l % mi;
            s += ainv[(long long)k * n + l] * b[(long long)I * C.rs + J];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) u[(long long)(1 + k / mi) * C.rs + 1 + k % mi] = s;
    }
}

// ---- 1D tridiagonal elimination (TridiagFactorization.solve, linalg.py:409-421) --------------
// One thread: the recurrence is sequential, and this keeps the reference's exact operation order.
__global__ void tri_solve_kernel(const double *__restrict__ b, double *__restrict__ x, int n,
                                 const double *__restrict__ sub, const double *__restrict__ dp,
                                 const double *__restrict__ cp, double *__restrict__ y) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    y[0] = b[0];
    for (int i = 1; i < n; ++i) y[i] = whb_sub(b[i], whb_mul(__ddiv_rn(sub[i - 1], dp[i - 1]), y[i - 1]));
    x[n - 1] = __ddiv_rn(y[n - 1], dp[n - 1]);
    for (int i = n - 2; i >= 0; --i) x[i] = whb_sub(__ddiv_rn(y[i], dp[i]), whb_mul(cp[i], x[i + 1]));
}

}  // namespace imp
