/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's explicit
 * WaveHoltz path (waveholtz 0.1.0, pure numpy).  Used by tests/ as the parity
 * checker where the numpy restatement is too slow, and by bench.py as the
 * multi-core CPU baseline.  Never linked into the product.
 *
 * Built with -O2 -ffp-contract=off (see oracle/Makefile) so every add/mul is a
 * separately rounded IEEE op in the same order as the reference's numpy
 * ufunc sequence; the results are therefore bitwise identical to
 * waveholtz.timestep.wave_solve_filtered (checked in tests/test_oracle_golden.py).
 *
 * Reference order:
 *   lap  = 0; for axis: lap += clo*w[-e]; lap += cmid*w; lap += clo*w[+e]   grid.py:357-365
 *   lap *= c2                                                               grid.py:366
 *   n==0: wn = w + half_dt2*(lap - f)                                       timestep.py:137
 *   n>0 : wn = (2*w - wp) + dt2*(lap - f*cos_f[n])                          timestep.py:139-140
 *   acc  = acc_c[0]*v (init), acc += acc_c[n+1]*wn                          timestep.py:284,298
 *   out  = out_scale*acc ; boundary = 0                                     timestep.py:300-301
 * Boundary (Dirichlet) points of w, f, v are exactly 0 and stay 0, so only
 * interior points are updated (boundary equivalence).
 *
 * Shapes are handled as 3D (n0,n1,n2) with the last `nd` axes active.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t n[3];
    int act[3];          /* axis active (has a stencil) */
    double clo[3], cmid[3];
    double c2;
} geom_t;

static void make_geom(geom_t *g, int nd, const int64_t *shape, const double *clo, const double *cmid,
                      double c2) {
    int off = 3 - nd;
    for (int a = 0; a < 3; ++a) {
        g->n[a] = 1;
        g->act[a] = 0;
        g->clo[a] = 0.0;
        g->cmid[a] = 0.0;
    }
    for (int a = 0; a < nd; ++a) {
        g->n[off + a] = shape[a];
        g->act[off + a] = 1;
        g->clo[off + a] = clo[a];
        g->cmid[off + a] = cmid[a];
    }
    g->c2 = c2;
}

/* kind: 0 first step, 1 middle step, 2 last step (writes out = s*(acc + cN*wN)) */
static void step(const geom_t *g, int kind, int zero_f, const double *w, const double *wp,
                 const double *f, double *wn, double *acc, double *out, double h, double cosn,
                 double acc0, double accn, double s, int use_c2, int nthreads) {
    const int64_t n0 = g->n[0], n1 = g->n[1], n2 = g->n[2];
    const int64_t s0 = n1 * n2, s1 = n2;
    const int64_t lo0 = g->act[0] ? 1 : 0, hi0 = g->act[0] ? n0 - 1 : 1;
    const int64_t lo1 = g->act[1] ? 1 : 0, hi1 = g->act[1] ? n1 - 1 : 1;
    const int64_t lo2 = 1, hi2 = n2 - 1;
    (void)nthreads;
#pragma omp parallel for collapse(2) schedule(static) num_threads(nthreads)
    for (int64_t i = lo0; i < hi0; ++i) {
        for (int64_t j = lo1; j < hi1; ++j) {
            for (int64_t k = lo2; k < hi2; ++k) {
                const int64_t p = i * s0 + j * s1 + k;
                const double wc = w[p];
                double lap = 0.0;
                if (g->act[0]) {
                    lap = lap + g->clo[0] * w[p - s0];
                    lap = lap + g->cmid[0] * wc;
                    lap = lap + g->clo[0] * w[p + s0];
                }
                if (g->act[1]) {
                    lap = lap + g->clo[1] * w[p - s1];
                    lap = lap + g->cmid[1] * wc;
                    lap = lap + g->clo[1] * w[p + s1];
                }
                lap = lap + g->clo[2] * w[p - 1];
                lap = lap + g->cmid[2] * wc;
                lap = lap + g->clo[2] * w[p + 1];
                if (use_c2) lap = lap * g->c2;
                double wnew;
                if (kind == 0) {
                    const double d = zero_f ? lap : lap - f[p];
                    wnew = wc + h * d;
                } else {
                    const double d = zero_f ? lap : lap - f[p] * cosn;
                    wnew = (2.0 * wc - wp[p]) + h * d;
                }
                if (kind == 0) {
                    wn[p] = wnew;
                    acc[p] = acc0 * wc + accn * wnew;
                } else if (kind == 1) {
                    wn[p] = wnew;
                    acc[p] = acc[p] + accn * wnew;
                } else {
                    out[p] = s * (acc[p] + accn * wnew);
                }
            }
        }
    }
}

static int64_t total(const int64_t *shape, int nd) {
    int64_t t = 1;
    for (int a = 0; a < nd; ++a) t *= shape[a];
    return t;
}

/* One application of W(v, f) (timestep.py:250-301, explicit).  out may alias v. */
int who_wave_solve(int nd, const int64_t *shape, const double *clo, const double *cmid, double c2,
                   const double *v, const double *f, int zero_f, int n_total, double half_dt2,
                   double dt2, const double *cos_f, const double *acc_c, double out_scale,
                   double *out, int nthreads) {
    if (nd < 1 || nd > 3 || n_total < 2) return -1;
    geom_t g;
    make_geom(&g, nd, shape, clo, cmid, c2);
    const int use_c2 = (c2 != 1.0);
    const int64_t N = total(shape, nd);
    double *b0 = (double *)calloc((size_t)N, sizeof(double));
    double *b1 = (double *)calloc((size_t)N, sizeof(double));
    double *b2 = (double *)calloc((size_t)N, sizeof(double));
    double *acc = (double *)calloc((size_t)N, sizeof(double));
    double *res = (double *)calloc((size_t)N, sizeof(double));
    if (!b0 || !b1 || !b2 || !acc || !res) {
        free(b0); free(b1); free(b2); free(acc); free(res);
        return -2;
    }
    /* w^0 = v (copy so out may alias v) */
    memcpy(b0, v, (size_t)N * sizeof(double));
    double *wm = b0, *wc = b1, *wn = b2;
    /* first step: w^1 into b1 */
    step(&g, 0, zero_f, b0, NULL, f, b1, acc, NULL, half_dt2, 1.0, acc_c[0], acc_c[1], 0.0,
         use_c2, nthreads);
    wm = b0;
    wc = b1;
    wn = b2;
    for (int n = 1; n < n_total; ++n) {
        const int last = (n == n_total - 1);
        step(&g, last ? 2 : 1, zero_f, wc, wm, f, wn, acc, res, dt2, cos_f[n], 0.0, acc_c[n + 1],
             out_scale, use_c2, nthreads);
        double *t = wm;
        wm = wc;
        wc = wn;
        wn = t;
    }
    memcpy(out, res, (size_t)N * sizeof(double));
    free(b0); free(b1); free(b2); free(acc); free(res);
    return 0;
}

/* FPI (driver.py:211-230): v0 = 0, `iters` passes of v <- W(v, f); resid[k] =
 * ||v_{k+1} - v_k||_2 / sqrt(N) (sum in index order; the reference uses BLAS
 * ddot, so residuals agree to rounding, iterates bitwise). */
int who_fpi(int nd, const int64_t *shape, const double *clo, const double *cmid, double c2,
            const double *f, int n_total, double half_dt2, double dt2, const double *cos_f,
            const double *acc_c, double out_scale, int iters, double *v, double *resid,
            int nthreads) {
    const int64_t N = total(shape, nd);
    double *vn = (double *)malloc((size_t)N * sizeof(double));
    if (!vn) return -2;
    memset(v, 0, (size_t)N * sizeof(double));
    for (int k = 0; k < iters; ++k) {
        int rc = who_wave_solve(nd, shape, clo, cmid, c2, v, f, 0, n_total, half_dt2, dt2, cos_f,
                                acc_c, out_scale, vn, nthreads);
        if (rc) { free(vn); return rc; }
        double ss = 0.0;
        for (int64_t p = 0; p < N; ++p) {
            const double d = vn[p] - v[p];
            ss += d * d;
        }
        resid[k] = sqrt(ss) / sqrt((double)N);
        memcpy(v, vn, (size_t)N * sizeof(double));
    }
    free(vn);
    return 0;
}

/* FPI with 5 resident fields (f, v, two time levels, acc) for grids whose
 * who_fpi working set (8 fields) does not fit host memory (1025^3 = 8.6 GB per
 * field).  Same per-point arithmetic and order as who_wave_solve: W^{n+1} is
 * written over W^{n-1} (each point reads only its own W^{n-1}), the last step
 * writes out = s*(acc + c_N W^N) over acc, and W^0 = v is read in place. */
int who_fpi_lean(int nd, const int64_t *shape, const double *clo, const double *cmid, double c2,
                 const double *f, int n_total, double half_dt2, double dt2, const double *cos_f,
                 const double *acc_c, double out_scale, int iters, double *v, double *resid,
                 int nthreads, int v_given) {
    if (nd < 1 || nd > 3 || n_total < 2) return -1;
    geom_t g;
    make_geom(&g, nd, shape, clo, cmid, c2);
    const int use_c2 = (c2 != 1.0);
    const int64_t N = total(shape, nd);
    double *wa = (double *)calloc((size_t)N, sizeof(double));
    double *wb = (double *)calloc((size_t)N, sizeof(double));
    double *acc = (double *)calloc((size_t)N, sizeof(double));
    if (!wa || !wb || !acc) {
        free(wa); free(wb); free(acc);
        return -2;
    }
    if (!v_given) memset(v, 0, (size_t)N * sizeof(double));  /* else continue from the caller's v */
    for (int k = 0; k < iters; ++k) {
        /* W^1 -> wa from W^0 = v */
        step(&g, 0, 0, v, NULL, f, wa, acc, NULL, half_dt2, 1.0, acc_c[0], acc_c[1], 0.0, use_c2,
             nthreads);
        /* W^2 -> wb (W^{n-1} = v is not overwritten) */
        double *wm = v, *wc = wa, *wn = wb;
        for (int n = 1; n < n_total; ++n) {
            const int last = (n == n_total - 1);
            step(&g, last ? 2 : 1, 0, wc, wm, f, wn, acc, acc, dt2, cos_f[n], 0.0, acc_c[n + 1],
                 out_scale, use_c2, nthreads);
            /* rotate; from n = 2 on the new level overwrites W^{n-1} in place */
            double *t = wc;
            wc = wn;
            wm = (n == 1) ? wa : t;
            wn = wm;
        }
        /* acc now holds v_new (boundary points: acc is 0 there).  The residual (a tolerance
         * quantity, not bitwise) is summed in long double: a sequential fp64 sum of 1e9 squares
         * drifts by ~1e-10 relative, more than the 1e-12 the GPU tests hold residuals to. */
        long double ss = 0.0L;
        for (int64_t p = 0; p < N; ++p) {
            const double d = acc[p] - v[p];
            ss += (long double)d * d;
        }
        resid[k] = sqrt((double)ss) / sqrt((double)N);
        memcpy(v, acc, (size_t)N * sizeof(double));
    }
    free(wa); free(wb); free(acc);
    return 0;
}

int who_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
