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
    // one block per row (plane, j); threads along the contiguous axis: no index divisions
    const long long nrows = (long long)(lp1 - lp0) * g.n1;
    for (long long row = blockIdx.x; row < nrows; row += gridDim.x) {
        const int plane = lp0 + (int)(row / g.n1);
        const int j = (int)(row - (long long)(plane - lp0) * g.n1);
        const bool row_in = (!A1 || (j >= g.j_lo && j < g.j_hi)) && (!A0 || (plane >= up0 && plane < up1));
        const long long base = (long long)plane * g.S0 + (long long)j * g.P;
        for (int k = threadIdx.x; k < g.n2; k += blockDim.x) {
            const long long p = base + k;
            const double xc = x[p];
            double lap = 0.0;
            if (row_in && k >= 1 && k < g.n2 - 1) {
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

// ---- device-resident CG scalars (cg_solve, linalg.py:62-99) -----------------------------------
// One CG iteration is enqueued as a fixed kernel sequence (capturable in a graph) whose
// scalars stay on the device: the host reads back p.Ap and r.r once per iteration, for the
// breakdown test and the convergence test the reference performs.
enum { CG_RZ = 0, CG_PAP = 1, CG_ALPHA = 2, CG_RR = 3, CG_RZN = 4, CG_BETA = 5, CG_NSC = 8 };

// finish a dot product (fixed-order tree) and derive the CG scalar that depends on it
__global__ void cg_final_kernel(const double *__restrict__ partials, int n, double *sc, int mode) {
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) t += partials[i];
    const double b = block_sum(t);
    if (threadIdx.x != 0) return;
    if (mode == 0) {         // p.Ap -> alpha = rz / pAp
        sc[CG_PAP] = b;
        sc[CG_ALPHA] = __ddiv_rn(sc[CG_RZ], b);
    } else if (mode == 1) {  // r.r
        sc[CG_RR] = b;
    } else if (mode == 2) {  // r.z (new) -> beta = rz_new / rz; rz = rz_new
        sc[CG_RZN] = b;
        sc[CG_BETA] = __ddiv_rn(b, sc[CG_RZ]);
        sc[CG_RZ] = b;
    } else {                 // initial r.z
        sc[CG_RZ] = b;
    }
}

__device__ __forceinline__ bool cg_ok(const double *sc) {
    const double pap = sc[CG_PAP];
    return pap > 0.0 && isfinite(pap);  // the reference stops on breakdown before updating x
}

// x = x + alpha*p; r = r - alpha*Ap
__global__ void cg_update_kernel(double *__restrict__ x, double *__restrict__ r, const double *__restrict__ p,
                                 const double *__restrict__ ap, const double *__restrict__ sc, long long n) {
    if (!cg_ok(sc)) return;
    const double a = sc[CG_ALPHA];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        x[i] = whb_add(x[i], whb_mul(a, p[i]));
        r[i] = whb_sub(r[i], whb_mul(a, ap[i]));
    }
}

// p = z + beta*p
__global__ void cg_dir_kernel(const double *__restrict__ z, double *__restrict__ p, const double *__restrict__ sc,
                              long long n) {
    if (!cg_ok(sc)) return;
    const double beta = sc[CG_BETA];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = whb_add(z[i], whb_mul(beta, p[i]));
}

// ---- 2D multigrid levels (linalg.py:189-283) -------------------------------------------------

struct Lev {
    int nx, ny;      // cells per axis (points nx+1, ny+1)
    long long rs;    // row stride (elements)
    double gx, gy, diag;
};

// one red-black colour: points with (i + j) % 2 == colour (linalg.py:230-238); one block per row
__global__ void gs_color_kernel(Lev L, double *__restrict__ u, const double *__restrict__ b, int color) {
    const int half = L.ny / 2 + 1;
    for (int i = 1 + blockIdx.x; i < L.nx; i += gridDim.x) {
        const int j0 = (i + color) & 1;
        const long long base = (long long)i * L.rs;
        for (int m = threadIdx.x; m < half; m += blockDim.x) {
            const int j = 2 * m + j0;
            if (j < 1 || j >= L.ny) continue;
            const long long p = base + j;
            const double v = whb_add(whb_add(b[p], whb_mul(L.gx, whb_add(u[p - L.rs], u[p + L.rs]))),
                                     whb_mul(L.gy, whb_add(u[p - 1], u[p + 1])));
            u[p] = __ddiv_rn(v, L.diag);
        }
    }
}

// H consecutive red-black half-sweeps (colours c0, 1-c0, c0, ...) in one pass: a CTA loads a
// (TY+2H) x (TX+2H) window of u and b into shared memory, applies half-sweep h on the window
// shrunk by h+1 cells (every value there depends only on window data), and writes back its
// TY x TX tile — the same arithmetic as H gs_color_kernel launches (temporal blocking of the
// smoother: one HBM pass and one launch instead of H).  Input and output are different arrays:
// neighbouring CTAs read their halos from `uin` while this one writes `uout`.
template <int TY, int TXW, int H>
__global__ void __launch_bounds__(256) gs_block_kernel(Lev L, const double *__restrict__ uin, double *__restrict__ uout,
                                                       const double *__restrict__ b, int c0) {
    constexpr int WR = TY + 2 * H, WC = TXW + 2 * H;
    __shared__ double su[WR * WC];
    __shared__ double sb[WR * WC];
    const int i0 = blockIdx.y * TY, j0 = blockIdx.x * TXW;  // tile origin (grid rows / columns)
    for (int t = threadIdx.x; t < WR * WC; t += blockDim.x) {
        const int wr = t / WC, wc = t - (t / WC) * WC;
        const int i = i0 - H + wr, j = j0 - H + wc;
        const bool in = i >= 0 && i <= L.nx && j >= 0 && j <= L.ny;
        const long long p = (long long)i * L.rs + j;
        su[t] = in ? uin[p] : 0.0;
        sb[t] = in ? b[p] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < H; ++h) {
        const int col = (c0 + h) & 1;
        const int m = h + 1;                    // margin: window cells not valid after this half-sweep
        const int nr = WR - 2 * m;              // rows updated
        const int nq = (WC - 2 * m + 1) / 2;    // colour points per row (upper bound)
        for (int t = threadIdx.x; t < nr * nq; t += blockDim.x) {
            const int wr = m + t / nq;
            const int i = i0 - H + wr;
            // first window column >= m whose grid column has the colour in this row
            const int wc = m + ((col - i - (j0 - H + m)) & 1) + 2 * (t - (t / nq) * nq);
            const int j = j0 - H + wc;
            if (wc >= WC - m || i < 1 || i >= L.nx || j < 1 || j >= L.ny) continue;
            const int w = wr * WC + wc;
            const double v = whb_add(whb_add(sb[w], whb_mul(L.gx, whb_add(su[w - WC], su[w + WC]))),
                                     whb_mul(L.gy, whb_add(su[w - 1], su[w + 1])));
            su[w] = __ddiv_rn(v, L.diag);
        }
        __syncthreads();
    }
    for (int t = threadIdx.x; t < TY * TXW; t += blockDim.x) {
        const int r = t / TXW, c = t - (t / TXW) * TXW;
        const int i = i0 + r, j = j0 + c;
        if (i >= 1 && i < L.nx && j >= 1 && j < L.ny) uout[(long long)i * L.rs + j] = su[(r + H) * WC + c + H];
    }
}

// Fused r = b - A u on the fine level + full-weighting restriction + zeroing of the coarse
// iterate: each coarse interior point forms the 9 fine residuals it weights (same values as
// residual_kernel; fine r is never stored) — one launch instead of three per level.
__device__ __forceinline__ double fine_resid(const Lev &F, const double *__restrict__ u, const double *__restrict__ b,
                                             long long p) {
    const double au = whb_sub(whb_sub(whb_mul(F.diag, u[p]), whb_mul(F.gx, whb_add(u[p - F.rs], u[p + F.rs]))),
                              whb_mul(F.gy, whb_add(u[p - 1], u[p + 1])));
    return whb_sub(b[p], au);
}

__global__ void resid_restrict_kernel(Lev F, const double *__restrict__ u, const double *__restrict__ b, Lev C,
                                      double *__restrict__ bc, double *__restrict__ uc) {
    for (int I = blockIdx.x; I <= C.nx; I += gridDim.x) {
        for (int J = threadIdx.x; J <= C.ny; J += blockDim.x) {
            double v = 0.0;
            if (I >= 1 && I < C.nx && J >= 1 && J < C.ny) {
                const long long p = (long long)(2 * I) * F.rs + 2 * J;
                const long long rs = F.rs;
                const double edges = whb_add(whb_add(whb_add(fine_resid(F, u, b, p - rs), fine_resid(F, u, b, p + rs)),
                                                     fine_resid(F, u, b, p - 1)),
                                             fine_resid(F, u, b, p + 1));
                const double corners =
                    whb_add(whb_add(whb_add(fine_resid(F, u, b, p - rs - 1), fine_resid(F, u, b, p - rs + 1)),
                                    fine_resid(F, u, b, p + rs - 1)),
                            fine_resid(F, u, b, p + rs + 1));
                v = __ddiv_rn(whb_add(whb_add(whb_mul(4.0, fine_resid(F, u, b, p)), whb_mul(2.0, edges)), corners),
                              16.0);
            }
            const long long q = (long long)I * C.rs + J;
            bc[q] = v;
            uc[q] = 0.0;
        }
    }
}

// u += prolong(ec) (bilinear, linalg.py:259-275, 337); one block per fine row
__global__ void prolong_add_kernel(Lev F, double *__restrict__ u, Lev C, const double *__restrict__ ec) {
    for (int i = blockIdx.x; i <= F.nx; i += gridDim.x) {
        const long long qrow = (long long)(i >> 1) * C.rs;
        const long long prow = (long long)i * F.rs;
        for (int j = threadIdx.x; j <= F.ny; j += blockDim.x) {
            const long long q = qrow + (j >> 1);
            double e;
            if (!(i & 1) && !(j & 1)) e = ec[q];
            else if ((i & 1) && !(j & 1)) e = whb_mul(0.5, whb_add(ec[q], ec[q + C.rs]));
            else if (!(i & 1) && (j & 1)) e = whb_mul(0.5, whb_add(ec[q], ec[q + 1]));
            else e = whb_mul(0.25, whb_add(whb_add(whb_add(ec[q], ec[q + C.rs]), ec[q + 1]), ec[q + C.rs + 1]));
            u[prow + j] = whb_add(u[prow + j], e);
        }
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

// ---- the coarse end of the V-cycle in ONE thread block ---------------------------------------
// Levels Lc..L-1 of a hierarchy are small (<= 65 x 65 points): their whole sub-cycle
// (smoothing, residual + restriction, coarse solve, prolongation, smoothing) runs in one CTA
// out of shared memory with block barriers between phases, instead of ~10 grid-wide launches
// per level whose cost is launch latency.  Same arithmetic as the per-level kernels above.
constexpr int kMaxCoarseLevels = 12;

struct CoarseCycle {
    Lev lev[kMaxCoarseLevels];  // levels Lc..L-1; rs = ny + 1 (compact in shared memory)
    int nlev, nu1, nu2;
    long long grs;              // row stride of level Lc's global arrays
};

__device__ __forceinline__ void cc_colour(const Lev &L, double *u, const double *b, int color) {
    const int half = L.ny / 2 + 1;
    const int total = (L.nx - 1) * half;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        const int i = 1 + t / half;
        const int j = 2 * (t - (i - 1) * half) + ((i + color) & 1);
        if (j < 1 || j >= L.ny) continue;
        const long long p = (long long)i * L.rs + j;
        const double v = whb_add(whb_add(b[p], whb_mul(L.gx, whb_add(u[p - L.rs], u[p + L.rs]))),
                                 whb_mul(L.gy, whb_add(u[p - 1], u[p + 1])));
        u[p] = __ddiv_rn(v, L.diag);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(1024) coarse_cycle_kernel(CoarseCycle cc, const double *__restrict__ gb,
                                                            double *__restrict__ gu, const double *__restrict__ ainv) {
    extern __shared__ __align__(16) double sm[];
    double *U[kMaxCoarseLevels], *B[kMaxCoarseLevels];
    {
        size_t off = 0;
        for (int l = 0; l < cc.nlev; ++l) {
            const size_t pts = (size_t)(cc.lev[l].nx + 1) * (cc.lev[l].ny + 1);
            U[l] = sm + off;
            off += pts;
            B[l] = sm + off;
            off += pts;
        }
    }
    {
        const Lev &L = cc.lev[0];
        const int total = (L.nx + 1) * (L.ny + 1);
        for (int t = threadIdx.x; t < total; t += blockDim.x) {
            const int i = t / (L.ny + 1), j = t - i * (L.ny + 1);
            B[0][t] = gb[(long long)i * cc.grs + j];
            U[0][t] = 0.0;
        }
        __syncthreads();
    }
    // down: pre-smooth, then r = b - A u restricted to the next level (its u = 0)
    for (int l = 0; l + 1 < cc.nlev; ++l) {
        const Lev &F = cc.lev[l];
        const Lev &C = cc.lev[l + 1];
        for (int k = 0; k < cc.nu1; ++k) {
            cc_colour(F, U[l], B[l], 0);
            cc_colour(F, U[l], B[l], 1);
        }
        const int total = (C.nx + 1) * (C.ny + 1);
        for (int t = threadIdx.x; t < total; t += blockDim.x) {
            const int I = t / (C.ny + 1), J = t - I * (C.ny + 1);
            double v = 0.0;
            if (I >= 1 && I < C.nx && J >= 1 && J < C.ny) {
                const long long p = (long long)(2 * I) * F.rs + 2 * J;
                const long long rs = F.rs;
                const double *u = U[l], *b = B[l];
                const double edges = whb_add(whb_add(whb_add(fine_resid(F, u, b, p - rs), fine_resid(F, u, b, p + rs)),
                                                     fine_resid(F, u, b, p - 1)),
                                             fine_resid(F, u, b, p + 1));
                const double corners =
                    whb_add(whb_add(whb_add(fine_resid(F, u, b, p - rs - 1), fine_resid(F, u, b, p - rs + 1)),
                                    fine_resid(F, u, b, p + rs - 1)),
                            fine_resid(F, u, b, p + rs + 1));
                v = __ddiv_rn(whb_add(whb_add(whb_mul(4.0, fine_resid(F, u, b, p)), whb_mul(2.0, edges)), corners),
                              16.0);
            }
            B[l + 1][t] = v;
            U[l + 1][t] = 0.0;
        }
        __syncthreads();
    }
    // coarsest: u = Ainv @ interior(b), one warp per unknown
    {
        const int c = cc.nlev - 1;
        const Lev &C = cc.lev[c];
        const int mi = C.ny - 1;
        const int n = (C.nx - 1) * mi;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
        for (int k = warp; k < n; k += nw) {
            double s = 0.0;
            for (int l2 = lane; l2 < n; l2 += 32) s += ainv[(long long)k * n + l2] * B[c][(1 + l2 / mi) * C.rs + 1 + l2 % mi];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) U[c][(1 + k / mi) * C.rs + 1 + k % mi] = s;
        }
        __syncthreads();
    }
    // up: u += prolong(e), post-smooth in reverse colour order
    for (int l = cc.nlev - 2; l >= 0; --l) {
        const Lev &F = cc.lev[l];
        const Lev &C = cc.lev[l + 1];
        const int total = (F.nx + 1) * (F.ny + 1);
        const double *ec = U[l + 1];
        for (int t = threadIdx.x; t < total; t += blockDim.x) {
            const int i = t / (F.ny + 1), j = t - i * (F.ny + 1);
            const long long q = (long long)(i >> 1) * C.rs + (j >> 1);
            double e;
            if (!(i & 1) && !(j & 1)) e = ec[q];
            else if ((i & 1) && !(j & 1)) e = whb_mul(0.5, whb_add(ec[q], ec[q + C.rs]));
            else if (!(i & 1) && (j & 1)) e = whb_mul(0.5, whb_add(ec[q], ec[q + 1]));
            else e = whb_mul(0.25, whb_add(whb_add(whb_add(ec[q], ec[q + C.rs]), ec[q + 1]), ec[q + C.rs + 1]));
            U[l][t] = whb_add(U[l][t], e);
        }
        __syncthreads();
        for (int k = 0; k < cc.nu2; ++k) {
            cc_colour(F, U[l], B[l], 1);
            cc_colour(F, U[l], B[l], 0);
        }
    }
    {
        const Lev &L = cc.lev[0];
        const int total = (L.nx + 1) * (L.ny + 1);
        for (int t = threadIdx.x; t < total; t += blockDim.x) {
            const int i = t / (L.ny + 1), j = t - i * (L.ny + 1);
            gu[(long long)i * cc.grs + j] = U[0][t];
        }
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
