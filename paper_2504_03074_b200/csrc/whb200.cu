// whb200 — B200-native (sm_100a) WaveHoltz explicit iteration: kernels + C ABI.
//
// One CUDA context object (whb_ctx) per (device, grid slab, batch of
// frequencies).  The hot path is ONE fused kernel per leapfrog step that, for
// every owned interior point, (a) applies the 3/5/7-point c^2*Laplacian,
// (b) advances the leapfrog update with forcing f*cos(w_e t^n), and (c) adds
// the trapezoidal filter term to the accumulator — so W^n is read once per
// step and never re-read for the filter.  The first
// step additionally initialises the accumulator; the last step applies the
// output scale and either writes the new iterate (plus the fixed-point
// residual partial sums), the plain filtered field, or the GMRES mat-vec
// x - W(x,0).
//
// Arithmetic order follows the reference exactly using
// explicitly rounded __dadd_rn/__dmul_rn (no FMA contraction), so every
// iterate is bitwise identical to waveholtz.timestep.wave_solve_filtered.
//
// Data layout in HBM: a field is stored as 3D
// (planes, n1, pitch) float64, planes = owned axis-0 planes + 2 x GH ghost planes,
// row pitch = n2 rounded up to 16 elements (128 B) so every row starts on a
// cache-line boundary.  2D grids (n0, n1) are stored as (n0, 1, n1) and 1D
// grids (n) as (1, 1, n), so the same kernel marches along storage axis 0
// with the contiguous axis across the warp.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include "nccl.h"

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <type_traits>
#include <tuple>
#include <vector>

#include "../../include/whb200.h"

namespace {

thread_local std::string g_last_error;

// ghost planes on each side of the owned planes: the two-step (temporal blocking) pass of a
// slab reads W^s two planes beyond its owned range
constexpr int GH = WHB_GHOST_PLANES;

int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

#define WHB_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t _e = (call);                                                                \
        if (_e != cudaSuccess)                                                                  \
            return fail(_e == cudaErrorMemoryAllocation ? WHB_E_NOMEM : WHB_E_CUDA,             \
                        std::string(#call) + ": " + cudaGetErrorString(_e));                    \
    } while (0)

#define WHB_TRY(expr)          \
    do {                       \
        int _rc = (expr);      \
        if (_rc) return _rc;   \
    } while (0)

// ------------------------------------------------------------------------------------------
// device-side descriptors

struct Geom {
    long long S0;     // plane stride (elements)
    int P;            // row pitch (elements)
    int n1, n2;       // extents of storage axes 1 and 2 (incl. boundary)
    int j_lo, j_hi;   // update range on axis 1 ([0,1) when axis 1 is degenerate)
    int i_lo, i_hi;   // local planes that are global-interior on axis 0 (owned or ghost)
    int use_c2;
    double clo0, cmid0, clo1, cmid1, clo2, cmid2, c2;
};

struct Member {
    double *v;              // W^0 / iterate
    const double *f;        // forcing or nullptr (zero forcing)
    double *ring[6];        // time level L >= 1 lives in ring[L mod nring] (level 0 = v)
    double *acc;            // filter accumulator
    double *dst;            // output of the last step (== v for FPI)
    const double *cos_f;    // [n_total]
    const double *acc_c;    // [n_total + 1]
    double half_dt2, dt2, out_scale;
    int n_total;
    int out_mode;
    double *partials;       // residual partial sums (FPI)
    int idx;                // member index (table order is by n_total, descending)
    int nring;              // 4 (passes of <= 2 steps) or 6 (passes of up to 4 steps)
};

enum { K_FIRST = 0, K_MID = 1, K_LAST = 2 };

// Buffer holding time level L of a member: W^0 is v, W^L (L >= 1) is ring[L mod nring].  A pass
// of T steps reads levels s, s-1 and writes s+T-1, s+T; the differences 1..T+1 never vanish
// mod nring when nring >= T+2 (4 slots for T <= 2, 6 slots for T <= 4), so no CTA of a pass
// ever overwrites a level another CTA of the same pass still reads.
__host__ __device__ __forceinline__ double *level_ptr(const Member &m, int L) {
    return L <= 0 ? m.v : m.ring[L % m.nring];
}

__device__ __forceinline__ double whb_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double whb_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double whb_mul(double a, double b) { return __dmul_rn(a, b); }

// Fused leapfrog + filter march over planes [i0, i1) of one (j, k) column.
template <int KIND, bool ZF, bool A0, bool A1>
__device__ __forceinline__ void march(const Geom &g, const Member &m, int s, int i0, int i1, int j,
                                      int k, double &rsum) {
    const double *__restrict__ wcur = level_ptr(m, s);
    const double *wprv = level_ptr(m, s - 1);
    double *wnxt = level_ptr(m, s + 1);  // never aliases levels s, s-1 (4-slot ring)
    const double *__restrict__ f = m.f;
    double *acc = m.acc;
    const double cosn = (KIND == K_FIRST) ? 1.0 : m.cos_f[s];
    const double h = (KIND == K_FIRST) ? m.half_dt2 : m.dt2;
    const double acc0 = m.acc_c[0];
    const double accn = m.acc_c[s + 1];
    const double sc = m.out_scale;
    const long long S0 = g.S0;
    const int P = g.P;

    long long p = (long long)i0 * S0 + (long long)j * P + k;
    double wm = A0 ? __ldg(wcur + p - S0) : 0.0;
    double wc = __ldg(wcur + p);
#pragma unroll 2
    for (int i = i0; i < i1; ++i, p += S0) {
        const double wp = A0 ? __ldg(wcur + p + S0) : 0.0;
        const double xl = __ldg(wcur + p - 1);
        const double xh = __ldg(wcur + p + 1);
        double yl = 0.0, yh = 0.0;
        if (A1) {
            yl = __ldg(wcur + p - P);
            yh = __ldg(wcur + p + P);
        }
        double fv = 0.0;
        if (!ZF) fv = __ldg(f + p);
        double wpv = 0.0;
        if (KIND != K_FIRST) wpv = wprv[p];
        double av = 0.0;
        if (KIND != K_FIRST) av = acc[p];

        // c^2 * Laplacian in reference order: out = 0; per axis: +lo, +mid, +hi (grid.py:357-366)
        double lap = 0.0;
        if (A0) {
            lap = whb_add(lap, whb_mul(g.clo0, wm));
            lap = whb_add(lap, whb_mul(g.cmid0, wc));
            lap = whb_add(lap, whb_mul(g.clo0, wp));
        }
        if (A1) {
            lap = whb_add(lap, whb_mul(g.clo1, yl));
            lap = whb_add(lap, whb_mul(g.cmid1, wc));
            lap = whb_add(lap, whb_mul(g.clo1, yh));
        }
        lap = whb_add(lap, whb_mul(g.clo2, xl));
        lap = whb_add(lap, whb_mul(g.cmid2, wc));
        lap = whb_add(lap, whb_mul(g.clo2, xh));
        if (g.use_c2) lap = whb_mul(lap, g.c2);

        double wn;
        if (KIND == K_FIRST) {
            // w1 = w + (dt^2/2)*(lap - f)                        timestep.py:137
            const double d = ZF ? lap : whb_sub(lap, fv);
            wn = whb_add(wc, whb_mul(h, d));
        } else {
            // w^{n+1} = (2w - w_prev) + dt^2*(lap - f*cos)       timestep.py:139-140
            const double d = ZF ? lap : whb_sub(lap, whb_mul(fv, cosn));
            wn = whb_add(whb_sub(whb_mul(2.0, wc), wpv), whb_mul(h, d));
        }
        if (KIND == K_FIRST) {
            // acc = c0*w0 ; acc += c1*w1                          timestep.py:284, 298
            wnxt[p] = wn;
            acc[p] = whb_add(whb_mul(acc0, wc), whb_mul(accn, wn));
        } else if (KIND == K_MID) {
            wnxt[p] = wn;
            acc[p] = whb_add(av, whb_mul(accn, wn));
        } else {
            const double out = whb_mul(sc, whb_add(av, whb_mul(accn, wn)));  // timestep.py:298-300
            if (m.out_mode == WHB_OUT_FPI) {
                const double vold = m.v[p];
                const double dd = out - vold;
                rsum += dd * dd;
                m.v[p] = out;
            } else if (m.out_mode == WHB_OUT_AV) {
                m.dst[p] = whb_sub(m.v[p], out);  // driver.py:259
            } else {
                m.dst[p] = out;
            }
        }
        wm = wc;
        wc = wp;
    }
}

template <int KIND, bool ZF, bool A0, bool A1>
__device__ __forceinline__ void march_guarded(const Geom &g, const Member &m, int s, int i0, int i1,
                                              int j, int k, bool act, double &rsum) {
    if (act) march<KIND, ZF, A0, A1>(g, m, s, i0, i1, j, k, rsum);
}

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    const int nw = (blockDim.x * blockDim.y + 31) >> 5;
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (tid < 32) {
        t = (tid < nw) ? red[tid] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    }
    return t;  // valid in thread 0
}

// One leapfrog step s for every active batch member (blockIdx.z).
// blockIdx.x: tile along the contiguous axis; blockIdx.y: (axis-1 tile, axis-0 chunk).
template <bool A0, bool A1>
__global__ void __launch_bounds__(256) step_kernel(Geom g, const Member *__restrict__ members, int s,
                                                   int i_begin, int i_end, int chunk_len, int JT,
                                                   int part_off) {
    const Member m = members[blockIdx.z];
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int jt = blockIdx.y % JT;
    const int ch = blockIdx.y / JT;
    const int j = A1 ? jt * blockDim.y + threadIdx.y : 0;
    const int i0 = i_begin + ch * chunk_len;
    const int i1 = min(i_end, i0 + chunk_len);
    const bool act = (k >= 1) && (k < g.n2 - 1) && (!A1 || (j >= g.j_lo && j < g.j_hi)) && (i0 < i1);
    const int kind = (s == 0) ? K_FIRST : ((s == m.n_total - 1) ? K_LAST : K_MID);
    const bool zf = (m.f == nullptr);
    double rsum = 0.0;
    if (kind == K_FIRST) {
        if (zf) march_guarded<K_FIRST, true, A0, A1>(g, m, s, i0, i1, j, k, act, rsum);
        else    march_guarded<K_FIRST, false, A0, A1>(g, m, s, i0, i1, j, k, act, rsum);
    } else if (kind == K_MID) {
        if (zf) march_guarded<K_MID, true, A0, A1>(g, m, s, i0, i1, j, k, act, rsum);
        else    march_guarded<K_MID, false, A0, A1>(g, m, s, i0, i1, j, k, act, rsum);
    } else {
        if (zf) march_guarded<K_LAST, true, A0, A1>(g, m, s, i0, i1, j, k, act, rsum);
        else    march_guarded<K_LAST, false, A0, A1>(g, m, s, i0, i1, j, k, act, rsum);
        if (m.out_mode == WHB_OUT_FPI) {
            const double t = block_sum(rsum);
            if (threadIdx.x == 0 && threadIdx.y == 0)
                m.partials[part_off + blockIdx.y * gridDim.x + blockIdx.x] = t;
        }
    }
}

// Deterministic residual reduction: hist[(*counter)*nb + b] = sum(partials_b[0:nparts]).
// The slots are zeroed as they are read: the last launch of the next pass (whose kernel, and so
// its number of partial sums, can differ after a schedule change) then only has to write its own.
__global__ void reduce_partials_kernel(const Member *__restrict__ members, int nb, int nparts,
                                       double *hist, int *counter) {
    __shared__ double red[32];
    const int slot = *counter;
    for (int b = 0; b < nb; ++b) {
        double *pp = members[b].partials;
        double t = 0.0;
        for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
            t += pp[i];
            pp[i] = 0.0;
        }
        for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
        __syncthreads();
        if (threadIdx.x < 32) {
            double u = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
            for (int o = 16; o > 0; o >>= 1) u += __shfl_down_sync(0xffffffffu, u, o);
            if (threadIdx.x == 0) hist[(long long)slot * nb + members[b].idx] = u;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *counter = slot + 1;
}

// Zero the Dirichlet boundary (and keep padding zero) of owned planes [lp0, lp1).
__global__ void zero_boundary_kernel(double *x, long long S0, int P, int n1, int n2, int act1,
                                     int lp0, int lp1, int zero_plane_lo, int zero_plane_hi, int per1, int per2) {
    const long long total = (long long)(lp1 - lp0) * S0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long pl = t / S0;
        const long long r = t - pl * S0;
        const int j = (int)(r / P);
        const int k = (int)(r - (long long)j * P);
        const int plane = lp0 + (int)pl;
        bool z = per2 ? (k >= n2) : ((k == 0) || (k >= n2 - 1));  // periodic axes have no boundary points
        if (act1 && !per1) z = z || (j == 0) || (j == n1 - 1);
        if (zero_plane_lo && plane == lp0) z = true;
        if (zero_plane_hi && plane == lp1 - 1) z = true;
        if (z) x[(long long)plane * S0 + r] = 0.0;
    }
}

}  // namespace
#include "step_bulk.cuh"
#include "step_tb2.cuh"
#include "step_t3.cuh"
#include "step_wf2d.cuh"
#include "step_cres2d.cuh"
#include "implicit.cuh"
namespace {

// y = c^2 * L_h x at owned interior points (DiscreteOperator.apply_values, grid.py:346-368);
// boundary and padding of y are left untouched (zero by invariant).
__global__ void apply_operator_kernel(Geom g, const double *__restrict__ x, double *__restrict__ y, int act0,
                                      int act1, int lp0, int lp1) {
    const long long total = (long long)(lp1 - lp0) * g.S0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long pl = t / g.S0;
        const long long r = t - pl * g.S0;
        const int j = (int)(r / g.P);
        const int k = (int)(r - (long long)j * g.P);
        if (k < 1 || k >= g.n2 - 1) continue;
        if (act1 && (j < g.j_lo || j >= g.j_hi)) continue;
        const long long p = (long long)(lp0 + pl) * g.S0 + r;
        const double wc = x[p];
        double lap = 0.0;
        if (act0) {
            lap = whb_add(lap, whb_mul(g.clo0, x[p - g.S0]));
            lap = whb_add(lap, whb_mul(g.cmid0, wc));
            lap = whb_add(lap, whb_mul(g.clo0, x[p + g.S0]));
        }
        if (act1) {
            lap = whb_add(lap, whb_mul(g.clo1, x[p - g.P]));
            lap = whb_add(lap, whb_mul(g.cmid1, wc));
            lap = whb_add(lap, whb_mul(g.clo1, x[p + g.P]));
        }
        lap = whb_add(lap, whb_mul(g.clo2, x[p - 1]));
        lap = whb_add(lap, whb_mul(g.cmid2, wc));
        lap = whb_add(lap, whb_mul(g.clo2, x[p + 1]));
        y[p] = whb_mul(lap, g.c2);  // out *= c**2 (grid.py:366)
    }
}

// ---- general operator: order p in {2, 4}, per-axis Dirichlet (odd reflection) or periodic
// (grid.py:296-306, 371-392).  One thread per point, LDG; every value
// is formed in the reference order (axis by axis, tap by tap from 0; reflected ghosts are
// the negated core value, multiplied like any other tap).
struct GeomG {
    long long S0;
    int P;
    int n[3];          // global extent of each storage axis
    int act[3];        // axis carries a stencil
    int per[3];        // periodic axis
    int order;         // 2 or 4
    int use_c2;
    int plane_begin;   // global index of local plane GH
    double taps[3][5];
    double c2;
};

// value of w at (global plane gi + o0, j + o1, k + o2) with boundary images; only one offset is nonzero
__device__ __forceinline__ double gfetch(const GeomG &g, const double *w, long long p, int gi, int j, int k, int axis,
                                         int o) {
    int idx = (axis == 0 ? gi : (axis == 1 ? j : k)) + o;
    const int n = g.n[axis];
    double sign = 1.0;
    if (g.per[axis]) {
        idx = (idx % n + n) % n;
    } else if (idx < 0) {
        idx = -idx;
        sign = -1.0;
    } else if (idx > n - 1) {
        idx = 2 * (n - 1) - idx;
        sign = -1.0;
    }
    long long q = p;
    if (axis == 0) q += (long long)(idx - gi) * g.S0;
    else if (axis == 1) q += (long long)(idx - j) * g.P;
    else q += (idx - k);
    const double v = w[q];
    return sign < 0.0 ? -v : v;
}

__device__ __forceinline__ double general_lap(const GeomG &g, const double *w, long long p, int gi, int j, int k) {
    const int h = g.order / 2;
    double lap = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (!g.act[a]) continue;
        for (int q = 0; q <= g.order; ++q) lap = whb_add(lap, whb_mul(g.taps[a][q], gfetch(g, w, p, gi, j, k, a, q - h)));
    }
    return g.use_c2 ? whb_mul(lap, g.c2) : lap;
}

__device__ __forceinline__ bool general_updates(const GeomG &g, int gi, int j, int k) {
    if (g.act[0] && !g.per[0] && (gi < 1 || gi > g.n[0] - 2)) return false;
    if (g.act[1] && !g.per[1] && (j < 1 || j > g.n[1] - 2)) return false;
    if (!g.per[2] && (k < 1 || k > g.n[2] - 2)) return false;
    return true;
}

// one leapfrog step for every active member (blockIdx.y), grid-stride over owned points
__global__ void step_general_kernel(GeomG g, const Member *__restrict__ members, int s, int nloc, int part_off) {
    const Member m = members[blockIdx.y];
    const int kind = (s == 0) ? K_FIRST : ((s == m.n_total - 1) ? K_LAST : K_MID);
    const double *wcur = level_ptr(m, s);
    const double *wprv = level_ptr(m, s - 1);
    double *wnxt = level_ptr(m, s + 1);
    const double cosn = (kind == K_FIRST) ? 1.0 : m.cos_f[s];
    const double h = (kind == K_FIRST) ? m.half_dt2 : m.dt2;
    const double acc0 = m.acc_c[0], accn = m.acc_c[s + 1];
    const int n1 = g.act[1] ? g.n[1] : 1, n2 = g.n[2];
    const long long total = (long long)nloc * n1 * n2;
    double rsum = 0.0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long pl = t / ((long long)n1 * n2);
        const long long r = t - pl * n1 * n2;
        const int j = (int)(r / n2);
        const int k = (int)(r - (long long)j * n2);
        const int gi = g.plane_begin + (int)pl;
        if (!general_updates(g, gi, j, k)) continue;
        const long long p = (pl + GH) * g.S0 + (long long)j * g.P + k;
        const double wc = wcur[p];
        const double lap = general_lap(g, wcur, p, gi, j, k);
        double wn;
        if (kind == K_FIRST) {
            const double d = m.f ? whb_sub(lap, m.f[p]) : lap;
            wn = whb_add(wc, whb_mul(h, d));
            wnxt[p] = wn;
            m.acc[p] = whb_add(whb_mul(acc0, wc), whb_mul(accn, wn));
        } else {
            const double d = m.f ? whb_sub(lap, whb_mul(m.f[p], cosn)) : lap;
            wn = whb_add(whb_sub(whb_mul(2.0, wc), wprv[p]), whb_mul(h, d));
            if (kind == K_MID) {
                wnxt[p] = wn;
                m.acc[p] = whb_add(m.acc[p], whb_mul(accn, wn));
            } else {
                const double out = whb_mul(m.out_scale, whb_add(m.acc[p], whb_mul(accn, wn)));
                if (m.out_mode == WHB_OUT_FPI) {
                    const double dd = out - m.v[p];
                    rsum += dd * dd;
                    m.v[p] = out;
                } else if (m.out_mode == WHB_OUT_AV) {
                    m.dst[p] = whb_sub(m.v[p], out);
                } else {
                    m.dst[p] = out;
                }
            }
        }
    }
    if (kind == K_LAST && m.out_mode == WHB_OUT_FPI) {
        const double b = block_sum(rsum);
        if (threadIdx.x == 0) m.partials[part_off + blockIdx.x] = b;
    }
}

#ifndef WHB_GM_MINB
#define WHB_GM_MINB 6  // resident blocks per SM the register allocation aims at
#endif
// One leapfrog step of the general operator, marching: thread = one (j, k) column of a chunk of
// axis-0 planes.  The 2h+1 axis-0 taps of the column come from a register window that takes one
// new (boundary-imaged) value per plane; axis-1/-2 taps are loads of neighbouring columns (L1 /
// L2 hits).  No 64-bit div/mod per point (the grid-stride kernel above decodes t -> (plane, j, k)).
// Whole-grid contexts only (plane_begin == 0), as the general plan.  Same arithmetic and order as
// general_lap / step_general_kernel.
template <int H>
__global__ void __launch_bounds__(128, WHB_GM_MINB) step_general_march_kernel(GeomG g, const Member *__restrict__ members,
                                                                              int s, int nloc, int chunk, int JY) {
    // (a reference, not a copy: level_ptr indexes the ring dynamically, which would put a copy of the
    // entry into every thread's local memory -- 160 B of stores per thread in blocks of 9 planes)
    const Member &m = members[blockIdx.z];
    const int kind = (s == 0) ? K_FIRST : ((s == m.n_total - 1) ? K_LAST : K_MID);
    const double *wcur = level_ptr(m, s);
    const double *wprv = level_ptr(m, s - 1);
    double *wnxt = level_ptr(m, s + 1);
    const double cosn = (kind == K_FIRST) ? 1.0 : m.cos_f[s];
    const double h = (kind == K_FIRST) ? m.half_dt2 : m.dt2;
    const double acc0 = m.acc_c[0], accn = m.acc_c[s + 1];
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y % JY;
    const int pl0 = (blockIdx.y / JY) * chunk;
    const int pl1 = min(nloc, pl0 + chunk);
    double rsum = 0.0;
    const bool col_ok = k < g.n[2];
    const long long cbase = (long long)j * g.P + k;  // column offset inside a plane
    // axis-0 window: win[q] = w at plane gi - H + q (imaged)
    double win[2 * H + 1];
    auto z_at = [&](int gi) -> double {  // w at global plane gi of this column, boundary-imaged
        int idx = gi;
        const int n = g.n[0];
        double sign = 1.0;
        if (g.per[0]) {
            idx = (idx % n + n) % n;
        } else if (idx < 0) {
            idx = -idx;
            sign = -1.0;
        } else if (idx > n - 1) {
            idx = 2 * (n - 1) - idx;
            sign = -1.0;
        }
        const double v = __ldg(wcur + (long long)(idx - g.plane_begin + GH) * g.S0 + cbase);
        return sign < 0.0 ? -v : v;
    };
    if (col_ok && pl0 < pl1 && g.act[0]) {
#pragma unroll
        for (int q = 0; q < 2 * H; ++q) win[q + 1] = z_at(g.plane_begin + pl0 - H + q);
    }
    // The operands of a plane that do not depend on the previous one -- the entering window value,
    // f, W^{n-1}, acc, v -- are loaded one iteration ahead: the stores of an iteration may alias the
    // next one's loads as far as the compiler knows, so without this every plane paid its DRAM round
    // trips in sequence (40.8 Gpts/s on the order-4 2049^2 workload, 0.28 of HBM).
    const double *const mf = m.f;
    double *const macc = m.acc, *const mv = m.v, *const mdst = m.dst;
    const int omode = m.out_mode;
    const double oscale = m.out_scale;
    const bool need_v = (kind == K_LAST) && omode != WHB_OUT_PLAIN;
    // (two planes ahead was measured slower: 40.0 vs 45.7 Gpts/s, one resident block less per SM)
    double zN = 0.0, fN = 0.0, pN = 0.0, aN = 0.0, vN = 0.0;
    // a chunk whose window stays inside the grid reads the entering value directly
    const bool zfast = g.per[0] == 0 && g.plane_begin + pl0 - H >= 0 && g.plane_begin + pl1 - 1 + H <= g.n[0] - 1;
    auto load_plane = [&](int pl) {
        if (g.act[0])
            zN = zfast ? __ldg(wcur + (long long)(pl + H + GH) * g.S0 + cbase) : z_at(g.plane_begin + pl + H);
        const long long p = (pl + GH) * g.S0 + cbase;
        if (mf) fN = mf[p];
        if (kind != K_FIRST) {
            pN = wprv[p];
            aN = macc[p];
        }
        if (need_v) vN = mv[p];
    };
    if (col_ok && pl0 < pl1) load_plane(pl0);
    // The axis-1 / axis-2 taps of a column sit at fixed offsets from the point (j and k do not change
    // along the march): boundary images (odd reflection / periodic wrap, as gfetch) are resolved
    // once per thread into an element offset and a sign per tap.
    long long off1[2 * H + 1], off2[2 * H + 1];
    bool neg1[2 * H + 1], neg2[2 * H + 1];
#pragma unroll
    for (int q = 0; q <= 2 * H; ++q) {
        auto image = [&](int axis, int c, long long stride, long long &off, bool &neg) {
            int idx = c + q - H;
            const int n = g.n[axis];
            neg = false;
            if (g.per[axis]) {
                idx = (idx % n + n) % n;
            } else if (idx < 0) {
                idx = -idx;
                neg = true;
            } else if (idx > n - 1) {
                idx = 2 * (n - 1) - idx;
                neg = true;
            }
            off = (long long)(idx - c) * stride;
        };
        image(1, j, g.P, off1[q], neg1[q]);
        image(2, k, 1, off2[q], neg2[q]);
    }
    // points of this column that are updated at all (axis-1 / axis-2 part of general_updates)
    const bool col_upd = col_ok && !(g.act[1] && !g.per[1] && (j < 1 || j > g.n[1] - 2)) &&
                         !(!g.per[2] && (k < 1 || k > g.n[2] - 2));
    const bool a0_bnd = g.act[0] && !g.per[0];
    for (int pl = pl0; pl < pl1 && col_ok; ++pl) {
        const int gi = g.plane_begin + pl;
        const double zc = zN, fc = fN, pc = pN, ac = aN, vc = vN;
        if (pl + 1 < pl1) load_plane(pl + 1);
        if (g.act[0]) {
#pragma unroll
            for (int q = 0; q < 2 * H; ++q) win[q] = win[q + 1];
            win[2 * H] = zc;
        }
        if (!col_upd || (a0_bnd && (gi < 1 || gi > g.n[0] - 2))) continue;
        const long long p = (pl + GH) * g.S0 + cbase;
        const double wc = g.act[0] ? win[H] : wcur[p];  // (an updated point is not a boundary image)
        double lap = 0.0;
        if (g.act[0]) {
#pragma unroll
            for (int q = 0; q <= 2 * H; ++q) lap = whb_add(lap, whb_mul(g.taps[0][q], win[q]));
        }
        if (g.act[1]) {
#pragma unroll
            for (int q = 0; q <= 2 * H; ++q) {
                const double v = wcur[p + off1[q]];
                lap = whb_add(lap, whb_mul(g.taps[1][q], neg1[q] ? -v : v));
            }
        }
        if (g.act[2]) {
#pragma unroll
            for (int q = 0; q <= 2 * H; ++q) {
                const double v = wcur[p + off2[q]];
                lap = whb_add(lap, whb_mul(g.taps[2][q], neg2[q] ? -v : v));
            }
        }
        if (g.use_c2) lap = whb_mul(lap, g.c2);
        double wn;
        if (kind == K_FIRST) {
            const double d = mf ? whb_sub(lap, fc) : lap;
            wn = whb_add(wc, whb_mul(h, d));
            wnxt[p] = wn;
            macc[p] = whb_add(whb_mul(acc0, wc), whb_mul(accn, wn));
        } else {
            const double d = mf ? whb_sub(lap, whb_mul(fc, cosn)) : lap;
            wn = whb_add(whb_sub(whb_mul(2.0, wc), pc), whb_mul(h, d));
            if (kind == K_MID) {
                wnxt[p] = wn;
                macc[p] = whb_add(ac, whb_mul(accn, wn));
            } else {
                const double out = whb_mul(oscale, whb_add(ac, whb_mul(accn, wn)));
                if (omode == WHB_OUT_FPI) {
                    const double dd = out - vc;
                    rsum += dd * dd;
                    mv[p] = out;
                } else if (omode == WHB_OUT_AV) {
                    mdst[p] = whb_sub(vc, out);
                } else {
                    mdst[p] = out;
                }
            }
        }
    }
    if (kind == K_LAST && m.out_mode == WHB_OUT_FPI) {
        const double b = block_sum(rsum);
        if (threadIdx.x == 0) m.partials[blockIdx.y * gridDim.x + blockIdx.x] = b;
    }
}

__global__ void apply_general_kernel(GeomG g, const double *__restrict__ x, double *__restrict__ y, int nloc) {
    const int n1 = g.act[1] ? g.n[1] : 1, n2 = g.n[2];
    const long long total = (long long)nloc * n1 * n2;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long pl = t / ((long long)n1 * n2);
        const long long r = t - pl * n1 * n2;
        const int j = (int)(r / n2);
        const int k = (int)(r - (long long)j * n2);
        const int gi = g.plane_begin + (int)pl;
        if (!general_updates(g, gi, j, k)) continue;
        const long long p = (pl + GH) * g.S0 + (long long)j * g.P + k;
        const int h = g.order / 2;
        double lap = 0.0;
        for (int a = 0; a < 3; ++a) {
            if (!g.act[a]) continue;
            for (int q = 0; q <= g.order; ++q) lap = whb_add(lap, whb_mul(g.taps[a][q], gfetch(g, x, p, gi, j, k, a, q - h)));
        }
        y[p] = whb_mul(lap, g.c2);  // out *= c**2 (grid.py:366)
    }
}

constexpr int kGenBlocks = 1184;

// Contiguous (rows, n) <-> pitched (rows, P): dir 1 scatters stage -> field, 0 gathers.
__global__ void repitch_kernel(double *stage, int n, double *field, int P, long long rows, int dir) {
    const long long total = rows * n;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t / n;
        const long long k = t - r * n;
        if (dir) field[r * P + k] = stage[t];
        else stage[t] = field[r * P + k];
    }
}

// Dirichlet boundary points and row padding of rows [ja, jb) of every owned plane := 0 (one thread
// per row: the two end segments, or the whole row on a boundary row / plane).
__global__ void band_zero_kernel(double *field, int n0, int n1, int n2, int P, long long S0, int ja, int jb) {
    const long long total = (long long)(jb - ja) * n0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int pl = (int)(t / (jb - ja));
        const int j = ja + (int)(t - (long long)pl * (jb - ja));
        double *row = field + pl * S0 + (long long)j * P;
        const bool whole = j == 0 || j == n1 - 1 || pl == 0 || pl == n0 - 1;
        row[0] = 0.0;
        for (int k = whole ? 1 : n2 - 1; k < P; ++k) row[k] = 0.0;
    }
}

// Write a scratch buffer larger than L2 so the next timed pass starts cold.
__global__ void l2_flush_kernel(double *buf, long long n, double val) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        buf[i] = val;
}

// ------------------------------------------------------------------------------------------
// vector kernels (owned planes only; padding and boundaries are zero in every vector)

constexpr int kRedBlocks = 592;  // 4 x 148 SMs; fixed => deterministic reduction order
constexpr int kRedThreads = 256;

__global__ void dot_partials_kernel(const double *__restrict__ x, const double *__restrict__ y,
                                    long long n, double *partials) {
    double t = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        t += x[i] * y[i];
    const double b = block_sum(t);
    if (threadIdx.x == 0) partials[blockIdx.x] = b;
}

__global__ void final_sum_kernel(const double *__restrict__ partials, int n, double *out) {
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) t += partials[i];
    const double b = block_sum(t);
    if (threadIdx.x == 0) *out = b;
}

// y -= h*x exactly as numpy's `w -= H[j,k]*Q[:,j]` (linalg.py:146): y = y - (h*x)
__global__ void axmy_kernel(double h, const double *__restrict__ x, double *y, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = __dsub_rn(y[i], __dmul_rn(h, x[i]));
}

__global__ void scale_kernel(double a, const double *__restrict__ x, double *y, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = __dmul_rn(x[i], a);
}

__global__ void div_kernel(const double *__restrict__ x, double d, double *y, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = __ddiv_rn(x[i], d);
}

// Modified Gram-Schmidt on the device (gmres_solve, linalg.py:143-150): one pass per basis
// vector applies the previous projection, w -= h[j-1] q[j-1] (h read from device memory), and
// forms the partial sums of the next coefficient q[j].w with the updated w — the same values,
// in the same order, as a separate axpy and dot (dot_partials_kernel's grid and order).
__global__ void mgs_step_kernel(double *__restrict__ w, const double *__restrict__ qprev,
                                const double *__restrict__ hprev, const double *__restrict__ q, long long n,
                                double *partials) {
    const double h = qprev ? *hprev : 0.0;
    double t = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double wi = w[i];
        if (qprev) {
            wi = __dsub_rn(wi, __dmul_rn(h, qprev[i]));
            w[i] = wi;
        }
        t += (q ? q[i] : wi) * wi;  // q == nullptr: w.w
    }
    const double b = block_sum(t);
    if (threadIdx.x == 0) partials[blockIdx.x] = b;
}

// q = w / sqrt(ww) when ww > 0 (Q[:, k+1] = w / ||w||, linalg.py:149-150)
__global__ void mgs_normalise_kernel(const double *__restrict__ w, const double *__restrict__ ww, double *q,
                                     long long n) {
    const double d2 = *ww;
    if (!(d2 > 0.0)) return;
    const double d = __dsqrt_rn(d2);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        q[i] = __ddiv_rn(w[i], d);
}

__global__ void sub_kernel(const double *__restrict__ x, const double *__restrict__ y, double *z,
                           long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        z[i] = __dsub_rn(x[i], y[i]);
}

constexpr int kMaxComb = 64;
struct CombArgs {
    const double *q[kMaxComb];
    double c[kMaxComb];
};

// y = y + sum_j c_j q_j (sum accumulated in j order, then added to y: x + Q@y, linalg.py:174)
__global__ void lincomb_kernel(CombArgs a, int count, double *y, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double t = 0.0;
        for (int jj = 0; jj < count; ++jj) t = __dadd_rn(t, __dmul_rn(a.q[jj][i], a.c[jj]));
        y[i] = __dadd_rn(y[i], t);
    }
}

}  // namespace

// ------------------------------------------------------------------------------------------
// host context

struct MemberHost {
    double *v = nullptr, *f = nullptr, *acc = nullptr, *out = nullptr;
    double *ring[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    double *cos_f = nullptr, *acc_c = nullptr, *partials = nullptr;
    std::vector<double> h_cos, h_acc;  // host copies (per-pass kernel parameters)
    double half_dt2 = 0, dt2 = 0, out_scale = 0;
    int n_total = 0;
};

namespace {
struct MGData;   // 2D multigrid hierarchy of the implicit solve (implicit.cuh)
struct TriData;  // 1D tridiagonal factorisation of the implicit solve
}  // namespace

struct whb_ctx {
    int device = 0;
    int ndim = 0;
    int64_t gshape[3] = {1, 1, 1};  // global storage shape (axis-0, axis-1, axis-2)
    int64_t plane_begin = 0, plane_end = 1;
    int64_t nloc = 1;               // owned planes
    int64_t nplanes = 1 + 2 * GH;   // allocated planes (owned + 2 x GH ghosts)
    int P = 16;
    int64_t S0 = 16;
    int64_t field_elems = 0;        // nplanes * S0
    int act0 = 0, act1 = 0;
    int nbatch = 1;
    int shared_f = 0;
    Geom geom{};
    bool op_set = false;
    cudaStream_t stream = nullptr;
    std::vector<MemberHost> mem;
    double *shared_f_ptr = nullptr;
    std::vector<double *> vecs;     // extra vectors (id 8 + i)
    Member *d_members = nullptr;    // device member table
    std::vector<Member> h_members;  // last uploaded
    std::vector<int> order;         // table order: members sorted by n_total desc
    double *d_hist = nullptr;
    int hist_cap = 0;
    int *d_counter = nullptr;
    double *d_red = nullptr;        // vector reduction scratch (kRedBlocks + 1)
    double *h_red = nullptr;        // pinned scalar
    double *d_mgs = nullptr, *h_mgs = nullptr;  // device / pinned MGS coefficients (whb_vec_mgs)
    int mgs_cap = 0;
    // launch geometry
    int kern = 1;                   // 1: TMA bulk-copy pipelined kernel (2D/3D), 0: simple LDG kernel
    size_t smem = 0;                // dynamic smem of the bulk kernel
    int64_t slack_front = 0, slack_back = 0;  // allocation slack around every field (bulk halo reads)
    int BX = 128, BY = 1, gx = 1, JT = 1, chunk_len = 1, nchunks = 1;
    int upd_lo = GH, upd_hi = GH + 1;  // local update planes [lo, hi)
    // two-step (temporal blocking) plan: whole-grid 2D/3D contexts
    bool tb2 = false;
    size_t smem2 = 0;
    int gx2 = 1, JT2 = 1, chunk2 = 1, nch2 = 1;
    // three-step (T = 3) plan: whole-grid single-problem 3D contexts (step_t3.cuh)
    bool t3 = false;
    size_t smem3 = 0;
    int gx3 = 1, JT3 = 1, JTE3 = 1, lxe3 = 32, chunk3 = 1, nch3 = 1;
    // row window of the next t3 / tb2 launches (the banded host iteration; whole grid: 0, INT_MAX, 0)
    int win_j0 = 0, win_j1 = INT_MAX, win_po = 0;
    int win_lxe = 0;  // edge tile shape of the windowed launches (0: lxe3)
    // cluster-resident small-grid 2D plan (whole grid in one cluster's shared memory)
    bool cres = false;
    int cres_cl = 0, cres_r = 0, cres_ppt = 1;
    // 2D wavefront plan (T steps per pass): whole-grid 2D contexts
    int wfT = 0;                     // 0 = off, else 2 or 4
    int nring = 4;                   // time-level buffers per member (6 for 3- and 4-step passes)
    int gxw[5] = {1, 1, 1, 1, 1}, chw[5] = {1, 1, 1, 1, 1}, nchw[5] = {1, 1, 1, 1, 1};
    long long wf_res[5] = {1, 1, 1, 1, 1};  // resident wavefront CTAs (SMs x CTAs per SM)
    size_t smemw[5] = {0, 0, 0, 0, 0};
    int nparts = 1;
    int64_t launches = 0;
    // graphs keyed by (out_mode, zf)
    std::map<std::tuple<int, int, const void *>, cudaGraphExec_t> graphs;
    std::map<std::tuple<int, int, const void *>, int64_t> graph_kernels;
    bool use_graphs = true;
    // timing
    bool timing = false;
    std::vector<cudaEvent_t> ev;
    // banded host iteration (whb_iterate_host on the three-step plan): copy-in / copy-out streams
    cudaStream_t s_in = nullptr, s_out = nullptr;
    std::vector<cudaStream_t> s_band;  // pass launches of band b go to s_band[b % size]
    std::vector<cudaEvent_t> ev_band;
    double t_step_ms = 0.0;
    int64_t t_step_launches = 0;
    double t_solve_ms = 0.0;
    // step-level (slab) solve state
    int cur_mode = -1, cur_zf = 0, cur_parts = 0;
    // optional L2 flush before every FPI pass (benchmark hygiene; not part of the timed span)
    double *flush_buf = nullptr;
    long long flush_elems = 0;
    double *stage = nullptr;         // contiguous staging buffer for host transfers
    GeomG geomg{};                   // general operator (kern == 3)
    int gm_gx = 0, gm_jy = 1, gm_chunk = 1, gm_nch = 0;  // its marching launch plan (0: grid-stride kernel)
    // TMA tensor maps keyed by (buffer, box kind)
    std::map<std::tuple<const double *, int, int>, CUtensorMap> tmaps;
    // implicit-mode solvers (whb_mg_setup / whb_tri_setup)
    MGData *mg = nullptr;
    TriData *tri = nullptr;
    double *d_cg = nullptr;          // device CG scalars (imp::CG_*)
    std::map<std::tuple<int, int, int, int, int, int, int, double>, cudaGraphExec_t> cg_graphs;
    // caller-captured graphs (whb_capture_begin/end): e.g. one slab iteration with its peer exchange
    bool capturing = false;
    std::vector<cudaGraphExec_t> user_graphs;
    // halo exchange stream: whb_comm_begin forks it from the context stream (event), copies / flag
    // writes / NCCL transfers issued until whb_comm_end go on it, whb_comm_join makes the context
    // stream wait for them -- so the interior planes enqueued in between overlap the exchange
    cudaStream_t comm = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool on_comm = false;
    // NCCL communicator of the slab ranks (whb_nccl_init), transfers on `comm`
    ncclComm_t nccl = nullptr;
    double *d_nccl = nullptr;  // all-reduce scratch
};

namespace {

struct MGLevelBuf {
    imp::Lev lev;
    double *u = nullptr, *b = nullptr, *r = nullptr;  // level 0: u/b are the caller's vectors
    double *raw[3] = {nullptr, nullptr, nullptr};      // owned allocations (coarse levels; r of level 0)
};

struct MGData {
    std::vector<MGLevelBuf> lv;
    int nu1 = 2, nu2 = 2;
    int lc = -1;               // first level of the single-CTA coarse sub-cycle (-1: none)
    size_t cc_smem = 0;
    imp::CoarseCycle cc{};
    double *ainv = nullptr;  // coarsest-level inverse, n x n
    std::map<std::pair<const double *, const double *>, cudaGraphExec_t> graphs;
};

struct TriData {
    int n = 0;
    double *sub = nullptr, *dp = nullptr, *cp = nullptr, *y = nullptr;
};

void free_mg(whb_ctx *c);
void free_tri(whb_ctx *c);

// Caller-captured graphs bake buffer pointers (d_hist, the schedule arrays, MG levels): when any of
// them is reallocated the graphs are destroyed and their ids stay invalid (whb_graph_launch then
// fails with WHB_E_STATE) until the caller captures again.
void invalidate_user_graphs(whb_ctx *c) {
    for (auto &ge : c->user_graphs)
        if (ge) {
            cudaGraphExecDestroy(ge);
            ge = nullptr;
        }
}

// CG iteration graphs bake the multigrid / tridiagonal buffers of the current setup
void drop_cg_graphs(whb_ctx *c) {
    for (auto &kv : c->cg_graphs) cudaGraphExecDestroy(kv.second);
    c->cg_graphs.clear();
}

int set_dev(whb_ctx *c) {
    WHB_CUDA(cudaSetDevice(c->device));
    return 0;
}

double *field_ptr(whb_ctx *c, int field, int member) {
    MemberHost &m = c->mem[member];
    switch (field) {
        case WHB_V: return m.v;
        case WHB_F: return c->shared_f ? c->shared_f_ptr : m.f;
        case WHB_WA: return m.ring[1];
        case WHB_WB: return m.ring[2];
        case WHB_WC: return m.ring[3];
        case WHB_WD: return m.ring[0];
        case WHB_ACC: return m.acc;
        case WHB_OUT: return m.out;
        default: return nullptr;
    }
}

// Every field is allocated with slack before and after it: the bulk kernel's
// row-segment loads may touch up to two rows before plane 0 and a few rows
// after the last plane (values there only feed points that are never updated).
int alloc_field(whb_ctx *c, double **p) {
    const size_t total = (size_t)(c->slack_front + c->field_elems + c->slack_back);
    double *raw = nullptr;
    WHB_CUDA(cudaMalloc(&raw, total * sizeof(double)));
    WHB_CUDA(cudaMemsetAsync(raw, 0, total * sizeof(double), c->stream));
    *p = raw + c->slack_front;
    return 0;
}

void free_field(whb_ctx *c, double *p) {
    if (p) cudaFree(p - c->slack_front);
}

int ensure_out(whb_ctx *c, int member) {
    if (!c->mem[member].out) return alloc_field(c, &c->mem[member].out);
    return 0;
}

double *vec_ptr(whb_ctx *c, int id) {
    if (id >= 0 && id <= WHB_WD) return field_ptr(c, id, 0);
    const int e = id - 8;
    if (e >= 0 && e < (int)c->vecs.size()) return c->vecs[e];
    return nullptr;
}

// owned region [plane GH, plane nloc+GH) of a field, as a flat element range
inline double *owned(double *base, whb_ctx *c) { return base + GH * c->S0; }
inline const double *owned(const double *base, whb_ctx *c) { return base + GH * c->S0; }
inline long long owned_elems(whb_ctx *c) { return (long long)c->nloc * c->S0; }

// Bulk-kernel tile configurations: 3D 8 x 64 tiles, 6 stages (17.7 KB each,
// 2 CTAs/SM); 2D 1 x 256 row segments, 8 stages (8.2 KB each, 3 CTAs/SM).
constexpr int B3_TX = 64, B3_BY = 8, B3_ST = 6;
constexpr int B2_TX = 256, B2_BY = 1, B2_ST = 8;

// Two-step kernel configurations: 3D 16 x 64 tiles, 5 stages (1 CTA/SM, 512 threads);
// 2D 256-column row strips, 8 stages (3 CTAs/SM).
constexpr int T3_TX = 64, T3_BY = 16, T3_ST = 5;  // measured on 257^3: BY = 8 / 4 stages / 2 CTAs per SM -0.6 %, BY = 12 / 6 stages -6 %
constexpr int T2_TX = 256, T2_BY = 1, T2_ST = 8;

template <bool A1, int K1, int K2, bool ZF, int GM = 0>
auto tb2_fn() {
    if constexpr (A1) return tb2::tb2_kernel<T3_TX, T3_BY, T3_ST, true, K1, K2, ZF, true, GM>;
    else return tb2::tb2_kernel<T2_TX, T2_BY, T2_ST, false, K1, K2, ZF, false, GM>;
}

// geometry mode of a context (wf2d / tb2 GM): equal taps on every active axis -> 1, and c^2 == 1 -> 2
int geom_mode(const whb_ctx *c) {
    const Geom &g = c->geom;
    const bool sq = c->act0 && g.clo0 == g.clo2 && g.cmid0 == g.cmid2 &&
                    (!c->act1 || (g.clo1 == g.clo0 && g.cmid1 == g.cmid0));
    return sq ? (g.use_c2 ? 1 : 2) : 0;
}

template <bool A1>
cudaError_t tb2_set_attrs(size_t smem) {
    cudaError_t e = cudaSuccess;
    auto set = [&](auto fn) {
        cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (r != cudaSuccess) e = r;
    };
    auto set_gm = [&](auto gm) {
        constexpr int GM = decltype(gm)::value;
        set(tb2_fn<A1, K_FIRST, K_MID, false, GM>()); set(tb2_fn<A1, K_FIRST, K_MID, true, GM>());
        set(tb2_fn<A1, K_MID, K_MID, false, GM>());   set(tb2_fn<A1, K_MID, K_MID, true, GM>());
        set(tb2_fn<A1, K_MID, K_LAST, false, GM>());  set(tb2_fn<A1, K_MID, K_LAST, true, GM>());
        set(tb2_fn<A1, K_FIRST, K_LAST, false, GM>()); set(tb2_fn<A1, K_FIRST, K_LAST, true, GM>());
    };
    set_gm(std::integral_constant<int, 0>{});
    set_gm(std::integral_constant<int, 1>{});
    set_gm(std::integral_constant<int, 2>{});
    return e;
}

// Three-step 3D kernel (step_t3.cuh): 6 TMA stages of 26 KB + the level-1/2 rings (206-225 KB), 1 CTA/SM.
#ifndef WHB_S3_ST
#define WHB_S3_ST 5
#endif
constexpr int S3_ST = WHB_S3_ST;
constexpr int S3_THREADS = t3::NTHREADS;

// LXE: tile shape of the last (ragged) column of tiles, t3::edge_lx(remaining columns)
template <int K1, int K2, bool ZF, int GM, int LXE>
auto t3_fn() {
    return t3::t3_kernel<S3_ST, K1, K2, ZF, GM, LXE>;
}

size_t t3_smem(int lxe) {
    return lxe == 4 ? t3::smem_bytes<S3_ST, 4>() : lxe == 8 ? t3::smem_bytes<S3_ST, 8>()
         : lxe == 16 ? t3::smem_bytes<S3_ST, 16>() : t3::smem_bytes<S3_ST, 32>();
}

// calls fn(integral_constant<int, LXE>) for the runtime shape
template <class F>
void t3_by_lxe(int lxe, F &&fn) {
    if (lxe == 4) fn(std::integral_constant<int, 4>{});
    else if (lxe == 8) fn(std::integral_constant<int, 8>{});
    else if (lxe == 16) fn(std::integral_constant<int, 16>{});
    else fn(std::integral_constant<int, 32>{});
}

cudaError_t t3_set_attrs(int lxe, size_t smem) {
    cudaError_t e = cudaSuccess;
    auto set = [&](auto fn) {
        cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (r != cudaSuccess) e = r;
    };
    t3_by_lxe(lxe, [&](auto lx) {
        constexpr int LXE = decltype(lx)::value;
        auto set_gm = [&](auto gm) {
            constexpr int GM = decltype(gm)::value;
            // (K_FIRST, K_LAST) is never launched: a 3-step solve would write v while reading it as W^0
            set(t3_fn<K_FIRST, K_MID, false, GM, LXE>()); set(t3_fn<K_FIRST, K_MID, true, GM, LXE>());
            set(t3_fn<K_MID, K_MID, false, GM, LXE>());   set(t3_fn<K_MID, K_MID, true, GM, LXE>());
            set(t3_fn<K_MID, K_LAST, false, GM, LXE>());  set(t3_fn<K_MID, K_LAST, true, GM, LXE>());
        };
        set_gm(std::integral_constant<int, 0>{});
        set_gm(std::integral_constant<int, 1>{});
        set_gm(std::integral_constant<int, 2>{});
    });
    return e;
}

// 2D wavefront kernels: 4 consumer warps + 1 producer warp, T + 4 row stages.
// (the WHB_WF_* macros exist for variant builds in tuning sweeps: tools/variants.py)
#ifndef WHB_WF_NW
#define WHB_WF_NW 4
#endif
#ifndef WHB_WF_ST_EXTRA
#define WHB_WF_ST_EXTRA 5
#endif
constexpr int WF_NW = WHB_WF_NW;

constexpr int WF_ST4 = 4 + WHB_WF_ST_EXTRA;  // 9 stages, 3 CTAs/SM (measured: 7 stages at 4 CTAs/SM is 1.4 % slower)
template <int T, int K1, int K2, bool ZF, bool PS = false, int GM = 0>
auto wf_fn() {
    if constexpr (T == 4) return wf2d::wf2d_kernel<4, WF_NW, WF_ST4, K1, K2, ZF, PS, GM>;
    else return wf2d::wf2d_kernel<T, WF_NW, T + 4, K1, K2, ZF, PS, GM>;
}

template <int T>
cudaError_t wf_set_attrs(size_t smem) {
    cudaError_t e = cudaSuccess;
    auto set = [&](auto fn) {
        cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (r != cudaSuccess) e = r;
    };
    auto set_gm = [&](auto ps, auto gm) {
        constexpr bool PS = decltype(ps)::value;
        constexpr int GM = decltype(gm)::value;
        set(wf_fn<T, K_FIRST, K_MID, false, PS, GM>()); set(wf_fn<T, K_FIRST, K_MID, true, PS, GM>());
        set(wf_fn<T, K_MID, K_MID, false, PS, GM>());   set(wf_fn<T, K_MID, K_MID, true, PS, GM>());
        set(wf_fn<T, K_MID, K_LAST, false, PS, GM>());  set(wf_fn<T, K_MID, K_LAST, true, PS, GM>());
        set(wf_fn<T, K_FIRST, K_LAST, false, PS, GM>()); set(wf_fn<T, K_FIRST, K_LAST, true, PS, GM>());
    };
    using F = std::false_type;
    using Tr = std::true_type;
    using G0 = std::integral_constant<int, 0>;
    using G1 = std::integral_constant<int, 1>;
    using G2 = std::integral_constant<int, 2>;
    set_gm(F{}, G0{}); set_gm(F{}, G1{}); set_gm(F{}, G2{});
    set_gm(Tr{}, G0{}); set_gm(Tr{}, G1{}); set_gm(Tr{}, G2{});
    return e;
}

template <bool A1, int KIND, bool ZF, bool TENSOR>
auto bulk_fn() {
    if constexpr (A1) return bulk::step_bulk_kernel<B3_TX, B3_BY, B3_ST, true, KIND, ZF, TENSOR>;
    else return bulk::step_bulk_kernel<B2_TX, B2_BY, B2_ST, false, KIND, ZF, false>;
}

template <bool A1, bool TENSOR>
cudaError_t bulk_set_attrs(size_t smem) {
    cudaError_t e = cudaSuccess;
    auto set = [&](auto fn) {
        cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (r != cudaSuccess) e = r;
    };
    set(bulk_fn<A1, K_FIRST, false, TENSOR>()); set(bulk_fn<A1, K_FIRST, true, TENSOR>());
    set(bulk_fn<A1, K_MID, false, TENSOR>());   set(bulk_fn<A1, K_MID, true, TENSOR>());
    set(bulk_fn<A1, K_LAST, false, TENSOR>());  set(bulk_fn<A1, K_LAST, true, TENSOR>());
    return e;
}

// ---- TMA tensor maps (3D path) --------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int get_encoder() {
    if (g_encode) return 0;
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
        return fail(WHB_E_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    return 0;
}

// ---- cluster-resident small-grid 2D kernel (step_cres2d.cuh) --------------------------------
constexpr size_t kCresSmemMax = 227 * 1024 - 1024;  // opt-in maximum less the static block_sum scratch

template <bool ZF, int GM, int PPT>
auto cres_fn() {
    return cres::cres2d_kernel<ZF, GM, PPT>;
}

cudaError_t cres_set_attrs() {
    cudaError_t e = cudaSuccess;
    auto set = [&](auto fn) {
        cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCresSmemMax);
        if (r != cudaSuccess) e = r;
        r = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (r != cudaSuccess) e = r;
    };
#define WHB_CRES_SET(PPT)                                                  \
    set(cres_fn<false, 0, PPT>()); set(cres_fn<true, 0, PPT>());           \
    set(cres_fn<false, 1, PPT>()); set(cres_fn<true, 1, PPT>());           \
    set(cres_fn<false, 2, PPT>()); set(cres_fn<true, 2, PPT>());
    WHB_CRES_SET(1) WHB_CRES_SET(2) WHB_CRES_SET(4) WHB_CRES_SET(8)
#undef WHB_CRES_SET
    return e;
}

// points per thread of a cluster of cl CTAs on this grid (0: more than cres::MAX_PPT)
int cres_ppt(whb_ctx *c, int cl) {
    const int NR = (int)c->gshape[0] - 2;
    const long long pts = (long long)((NR + cl - 1) / cl) * (c->gshape[2] - 2);
    for (int p = 1; p <= cres::MAX_PPT; p *= 2)
        if (pts <= (long long)p * cres::NT) return p;
    return 0;
}

int cres_max_clusters(whb_ctx *c, int cl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl, 1, 1);
    cfg.blockDim = dim3(cres::NT, 1, 1);
    const int R = ((int)c->gshape[0] - 2 + cl - 1) / cl;
    cfg.dynamicSmemBytes = cres::smem_doubles(R, (int)c->gshape[2], 64, cl) * sizeof(double);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, cres_fn<false, 0, 8>(), &cfg);
    if (e != cudaSuccess) {
        if (getenv("WHB_DEBUG")) fprintf(stderr, "[whb] cudaOccupancyMaxActiveClusters: %s\n", cudaGetErrorString(e));
        cudaGetLastError();
        n = 0;
    }
    return n;
}

int occupancy_blocks(whb_ctx *c) {
    int nb = 0;
    cudaError_t e;
    const int threads = c->BX * c->BY;
    if (c->kern == 1) {
        if (c->act1) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bulk_fn<true, K_MID, false, true>(), B3_TX * B3_BY / 2, c->smem);
        else e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bulk_fn<false, K_MID, false, false>(), B2_TX * B2_BY / 2, c->smem);
    } else if (c->act1) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, step_kernel<true, true>, threads, 0);
    else if (c->act0) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, step_kernel<true, false>, threads, 0);
    else e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, step_kernel<false, false>, threads, 0);
    if (e != cudaSuccess || nb < 1) nb = 1;
    return nb;
}

int plan_launch(whb_ctx *c) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    const char *kenv = getenv("WHB_KERNEL");
    const std::string kname = kenv ? kenv : "";
    // 3D single problem: TMA tensor boxes (kern 2); 2D / batched: per-row bulk copies (kern 1)
    c->kern = !c->act0 ? 0 : (kname == "simple" ? 0 : ((c->act1 && c->nbatch == 1 && kname != "bulk") ? 2 : 1));
    if (c->kern == 2) WHB_TRY(get_encoder());
    if (c->kern >= 1) {
        c->BX = c->act1 ? B3_TX : B2_TX;
        c->BY = c->act1 ? B3_BY : B2_BY;
        c->smem = c->act1 ? bulk::bulk_smem_bytes<B3_TX, B3_BY, B3_ST, true>()
                          : bulk::bulk_smem_bytes<B2_TX, B2_BY, B2_ST, false>();
        cudaError_t e = c->act1 ? (c->kern == 2 ? bulk_set_attrs<true, true>(c->smem) : bulk_set_attrs<true, false>(c->smem))
                                : bulk_set_attrs<false, false>(c->smem);
        if (e != cudaSuccess) return fail(WHB_E_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    } else {
        c->BX = c->act1 ? 32 : 128;
        c->BY = c->act1 ? 8 : 1;
        c->smem = 0;
    }
    const int64_t n1 = c->gshape[1], n2 = c->gshape[2];
    c->gx = (int)((n2 - 1 + c->BX - 1) / c->BX);               // covers k in [0, n2-1)
    c->JT = c->act1 ? (int)((n1 - 1 + c->BY - 1) / c->BY) : 1;  // covers j in [0, n1-1)
    // local update planes: owned planes that are global-interior along axis 0
    if (c->act0) {
        const int64_t g_lo = std::max<int64_t>(c->plane_begin, 1);
        const int64_t g_hi = std::min<int64_t>(c->plane_end, c->gshape[0] - 1);
        c->upd_lo = (int)(g_lo - c->plane_begin + GH);
        c->upd_hi = (int)std::max<int64_t>(g_hi - c->plane_begin + GH, c->upd_lo);
    } else {
        c->upd_lo = GH;
        c->upd_hi = GH + 1;
    }
    const int nplanes = std::max(1, c->upd_hi - c->upd_lo);
    const int per_sm = occupancy_blocks(c);
    const long long resident = (long long)sms * per_sm;
    const long long tiles = (long long)c->gx * c->JT;
    int cl;
    if (c->kern >= 1) {
        // marching kernel: 2D -> one wave of long-lived CTAs; 3D -> ~4 waves (measured: 257^3
        // 1 wave 101.6, 2 waves 109.0, 3.5 waves 111.4 Gpts/s); chunk only when tiles are scarce
        const long long waves = c->act1 ? 4 : 1;
        const long long nch = std::max<long long>(1, waves * resident / std::max<long long>(1, tiles));
        cl = (int)((nplanes + nch - 1) / nch);
    } else {
        const long long target = resident * 2;
        int nch = (int)std::max<long long>(1, target / std::max<long long>(1, tiles));
        cl = (nplanes + nch - 1) / nch;
        const int min_chunk = c->act1 ? 4 : 8;
        if (cl < min_chunk) cl = std::min(nplanes, min_chunk);
    }
    const char *env = getenv("WHB_CHUNK");
    if (env && atoi(env) > 0) cl = atoi(env);
    if (!c->act0) cl = 1;
    c->chunk_len = std::max(1, cl);
    c->nchunks = (nplanes + c->chunk_len - 1) / c->chunk_len;
    if ((long long)c->JT * c->nchunks > 65535)
        return fail(WHB_E_ARG, "grid too large for launch plan (axis-1 tiles x chunks > 65535)");
    c->nparts = c->gx * c->JT * (c->nchunks + 2);
    // two-step plan: 2D/3D contexts, whole grids and slabs (GH = 2 ghost planes per side feed the
    // pass); WHB_TB2=0 keeps one step per pass
    const char *tenv = getenv("WHB_TB2");
    const bool whole = c->plane_begin == 0 && c->plane_end == c->gshape[0];
    c->tb2 = c->kern >= 1 && c->act0 && !(tenv && std::string(tenv) == "0") && (!c->act1 || c->kern == 2) &&
             c->upd_hi - c->upd_lo >= 1;
    if (c->tb2) {
        const int TX = c->act1 ? T3_TX : T2_TX, BYt = c->act1 ? T3_BY : T2_BY;
        c->smem2 = c->act1 ? tb2::tb2_smem_bytes<T3_TX, T3_BY, T3_ST, true>()
                           : tb2::tb2_smem_bytes<T2_TX, T2_BY, T2_ST, false>();
        cudaError_t e = c->act1 ? tb2_set_attrs<true>(c->smem2) : tb2_set_attrs<false>(c->smem2);
        if (e != cudaSuccess) return fail(WHB_E_CUDA, std::string("cudaFuncSetAttribute(tb2): ") + cudaGetErrorString(e));
        int nb = 0;
        if (c->act1) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, tb2_fn<true, K_MID, K_MID, false>(), TX * BYt / 2, c->smem2);
        else e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, tb2_fn<false, K_MID, K_MID, false>(), TX * BYt / 2, c->smem2);
        if (e != cudaSuccess || nb < 1) return fail(WHB_E_CUDA, "tb2 kernel does not fit on an SM");
        c->gx2 = (int)((n2 - 1 + TX - 1) / TX);
        c->JT2 = c->act1 ? (int)((n1 - 1 + BYt - 1) / BYt) : 1;
        const long long res2 = (long long)sms * nb;
        const long long tiles2 = (long long)c->gx2 * c->JT2;
        const long long waves = c->act1 ? 4 : 1;
        const long long nch = std::max<long long>(1, waves * res2 / std::max<long long>(1, tiles2));
        int cl2 = (int)((nplanes + nch - 1) / nch);
        const char *env2 = getenv("WHB_CHUNK2");
        if (env2 && atoi(env2) > 0) cl2 = atoi(env2);
        c->chunk2 = std::max(1, cl2);
        c->nch2 = (nplanes + c->chunk2 - 1) / c->chunk2;
        if ((long long)c->JT2 * c->nch2 > 65535) c->tb2 = false;
        c->nparts = std::max(c->nparts, c->gx2 * c->JT2 * (c->nch2 + 2));
    }
    // 2D wavefront plan (default for whole-grid 2D contexts; WHB_WF=0 disables, WHB_WF=2 picks T = 2)
    const char *wenv = getenv("WHB_WF");
    c->wfT = (c->tb2 && whole && !c->act1 && !(wenv && std::string(wenv) == "0")) ? ((wenv && std::string(wenv) == "2") ? 2 : 4) : 0;
    if (c->wfT) {
        for (int T : {2, 4}) {
            if (T > c->wfT) continue;
            const int CW = WF_NW * (64 - 2 * T);
            c->smemw[T] = T == 2 ? wf2d::wf_smem_bytes<2, WF_NW, 6>()
                                 : wf2d::wf_smem_bytes<4, WF_NW, WF_ST4>();
            cudaError_t e = T == 2 ? wf_set_attrs<2>(c->smemw[T]) : wf_set_attrs<4>(c->smemw[T]);
            if (e != cudaSuccess) return fail(WHB_E_CUDA, std::string("cudaFuncSetAttribute(wf): ") + cudaGetErrorString(e));
            int nb = 0;
            e = T == 2 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, wf_fn<2, K_MID, K_MID, false>(), 32 * (WF_NW + 1), c->smemw[T])
                       : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, wf_fn<4, K_MID, K_MID, false>(), 32 * (WF_NW + 1), c->smemw[T]);
            if (e != cudaSuccess || nb < 1) return fail(WHB_E_CUDA, "wavefront kernel does not fit on an SM");
            c->gxw[T] = (int)((n2 - 1 + CW - 1) / CW);
            const long long res = (long long)sms * nb;
            c->wf_res[T] = res;
            const long long nch = std::max<long long>(1, res / std::max<long long>(1, c->gxw[T]));
            int cl = (int)((nplanes + nch - 1) / nch);
            const char *ce = getenv("WHB_CHUNKW");
            if (ce && atoi(ce) > 0) cl = atoi(ce);
            c->chw[T] = std::max(1, cl);
            c->nchw[T] = (nplanes + c->chw[T] - 1) / c->chw[T];
            if (c->nchw[T] > 65535) c->wfT = 0;
            c->nparts = std::max(c->nparts, c->gxw[T] * (c->nchw[T] + 2));
        }
    }
    // three-step plan (default for whole-grid single-problem 3D contexts; WHB_T3=0 disables): output
    // tiles of 12 x 60 (t3::BY x t3::TX), axis-0 chunks of ~256 planes (a chunk re-streams 5 warm-up
    // planes); small grids whose tiles cannot fill the GPU with chunks of >= 48 planes keep tb2
    const char *t3env = getenv("WHB_T3");
    c->t3 = false;
    if (c->tb2 && c->act1 && c->kern == 2 && c->nbatch == 1 && !(t3env && std::string(t3env) == "0")) {
        // column tiles: full main tiles, then one tile of the narrowest shape covering the rest
        const int gfull = (int)((n2 - 1) / t3::TX);
        const int rem = (int)(n2 - 1) - gfull * t3::TX;
        const char *e3 = getenv("WHB_T3_EDGE");  // 0: main shape on the ragged edge too (A/B)
        c->lxe3 = (rem == 0 || (e3 && std::string(e3) == "0")) ? 32 : t3::edge_lx(rem);
        c->smem3 = t3_smem(c->lxe3);
        cudaError_t e = t3_set_attrs(c->lxe3, c->smem3);
        // (the banded host iteration picks a wider, shorter edge shape per band height)
        for (int lx = c->lxe3 * 2; lx <= 16 && c->lxe3 != 32 && e == cudaSuccess; lx *= 2) e = t3_set_attrs(lx, t3_smem(lx));
        if (e != cudaSuccess) return fail(WHB_E_CUDA, std::string("cudaFuncSetAttribute(t3): ") + cudaGetErrorString(e));
        int nb = 0;
        t3_by_lxe(c->lxe3, [&](auto lx) {
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, t3_fn<K_MID, K_MID, false, 2, decltype(lx)::value>(),
                                                              S3_THREADS, c->smem3);
        });
        if (e != cudaSuccess || nb < 1) return fail(WHB_E_CUDA, "t3 kernel does not fit on an SM");
        c->gx3 = gfull + (rem > 0 ? 1 : 0);
        c->JT3 = (int)((n1 - 1 + t3::BY - 1) / t3::BY);
        const int bye = c->lxe3 == 4 ? t3::Shape<4>::BY : c->lxe3 == 8 ? t3::Shape<8>::BY
                      : c->lxe3 == 16 ? t3::Shape<16>::BY : t3::BY;
        c->JTE3 = (int)((n1 - 1 + bye - 1) / bye);
        const long long tiles3 = (long long)c->gx3 * c->JT3;
        const long long res3 = (long long)sms * nb;
        // chunks: ~256 planes, but at least 2 waves of CTAs (measured, Gpts/s -- 257^3: chunks of 52 / 64 /
        // 86 / 128 / 255 planes 212 / 220 / 226 / 199 / 184, the two-step kernel 182; 1025^3: 256 / 342 /
        // 512 / 1023 planes 250 / 249 / 242 / 225)
        long long nch = std::max<long long>((nplanes + 255) / 256, (2 * res3 + tiles3 - 1) / tiles3);
        int cl3 = (int)((nplanes + nch - 1) / nch);
        const char *env3 = getenv("WHB_CHUNK3");
        if (env3 && atoi(env3) > 0) cl3 = atoi(env3);
        c->chunk3 = std::max(1, cl3);
        c->nch3 = (nplanes + c->chunk3 - 1) / c->chunk3;
        c->t3 = ((long long)c->JT3 * c->nch3 <= 65535) &&
                (c->chunk3 >= 48 || (t3env && std::string(t3env) == "1"));
        // (the banded host iteration launches one wave of CTAs per band of 12 rows and pass)
        if (c->t3) c->nparts = std::max(c->nparts, std::max(c->gx3 * c->JT3 * c->nch3, c->JT3 * 2 * sms));
    }
    c->nring = (c->wfT == 4 || c->t3) ? 6 : 4;
    // cluster-resident plan (whole-grid 2D with the fields in one cluster's shared memory; the
    // per-launch fit against the step count is cres_fits); WHB_CRES=0 disables, WHB_CRES_CL=n
    // caps the cluster size
    const char *cenv = getenv("WHB_CRES");
    c->cres = false;
    if (whole && c->act0 && !c->act1 && c->kern >= 1 && !(cenv && std::string(cenv) == "0")) {
        const int NR = (int)c->gshape[0] - 2;
        const char *clenv = getenv("WHB_CRES_CL");
        int cl = clenv && atoi(clenv) > 0 ? atoi(clenv) : cres::MAX_CL;
        cl = std::min(cl, cres::MAX_CL);
        while (cl > 1 && cl > NR) cl >>= 1;
        const int W = (int)c->gshape[2];
        const cudaError_t ae = NR >= 1 ? cres_set_attrs() : cudaErrorInvalidValue;
        if (getenv("WHB_DEBUG")) fprintf(stderr, "[whb] cres attrs: %s\n", cudaGetErrorString(ae));
        if (ae == cudaSuccess) {
            // the cluster must be schedulable (cl SMs of one GPC): fall back to smaller clusters
            for (; cl >= 1; cl >>= 1) {
                const int R = (NR + cl - 1) / cl;
                if (cres::smem_doubles(R, W, 64, cl) * sizeof(double) > kCresSmemMax || !cres_ppt(c, cl)) break;
                const int mc = cres_max_clusters(c, cl);
                if (getenv("WHB_DEBUG")) fprintf(stderr, "[whb] cres cluster %d: %d active clusters\n", cl, mc);
                if (mc > 0) {
                    c->cres = true;
                    c->cres_cl = cl;
                    c->cres_r = R;
                    c->cres_ppt = cres_ppt(c, cl);
                    break;
                }
            }
        }
        cudaGetLastError();
    }
    // slack: bulk row segments start 2 columns / 1 row early and may run BY+1 rows past the last plane
    c->slack_front = 2 * (int64_t)c->P + 32;
    c->slack_back = (int64_t)(c->BY + 3) * c->P + c->BX + 64;
    return 0;
}

int ensure_hist(whb_ctx *c, int iters) {
    if (iters <= c->hist_cap) return 0;
    if (c->d_hist) {
        WHB_CUDA(cudaStreamSynchronize(c->stream));
        WHB_CUDA(cudaFree(c->d_hist));
    }
    int cap = std::max(iters, 64);
    WHB_CUDA(cudaMalloc(&c->d_hist, (size_t)cap * c->nbatch * sizeof(double)));
    c->hist_cap = cap;
    // graphs bake the hist pointer
    for (auto &kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
    invalidate_user_graphs(c);
    return 0;
}

// Build the member table for a call and upload it if it changed.
int upload_members(whb_ctx *c, int out_mode, int zf, const double *vx = nullptr, double *dst = nullptr) {
    std::vector<Member> t(c->nbatch);
    for (int pos = 0; pos < c->nbatch; ++pos) {
        const int b = c->order[pos];
        MemberHost &h = c->mem[b];
        Member m{};
        m.v = vx ? const_cast<double *>(vx) : h.v;
        m.f = zf ? nullptr : (c->shared_f ? c->shared_f_ptr : h.f);
        for (int q = 0; q < 6; ++q) m.ring[q] = h.ring[q];
        m.nring = c->nring;
        m.acc = h.acc;
        if (out_mode == WHB_OUT_FPI) m.dst = m.v;
        else {
            if (dst) m.dst = dst;
            else {
                WHB_TRY(ensure_out(c, b));
                m.dst = h.out;
            }
        }
        m.cos_f = h.cos_f;
        m.acc_c = h.acc_c;
        m.half_dt2 = h.half_dt2;
        m.dt2 = h.dt2;
        m.out_scale = h.out_scale;
        m.n_total = h.n_total;
        m.out_mode = out_mode;
        m.partials = h.partials;
        m.idx = b;
        t[pos] = m;
    }
    bool same = c->h_members.size() == t.size() &&
                std::memcmp(c->h_members.data(), t.data(), t.size() * sizeof(Member)) == 0;
    if (!same) {
        // table is read by in-flight kernels: order the update on the stream
        WHB_CUDA(cudaMemcpyAsync(c->d_members, t.data(), t.size() * sizeof(Member),
                                 cudaMemcpyHostToDevice, c->stream));
        WHB_CUDA(cudaStreamSynchronize(c->stream));  // t is pageable & local
        c->h_members = t;
    }
    return 0;
}

struct StepMaps {
    CUtensorMap w, p, f, a;
};

template <bool A1, int KIND, bool ZF, bool TENSOR>
void launch_bulk(whb_ctx *c, dim3 grid, int member_off, int s, int i_begin, int i_end, int chunk_len, int part_off,
                 const StepMaps &mp) {
    constexpr int threads = A1 ? B3_TX * B3_BY / 2 : B2_TX * B2_BY / 2;
    bulk_fn<A1, KIND, ZF, TENSOR>()<<<grid, threads, c->smem, c->stream>>>(
        c->geom, c->d_members, member_off, s, i_begin, i_end, chunk_len, c->JT, part_off, mp.w, mp.p, mp.f, mp.a);
}

template <bool A1, bool TENSOR>
void launch_bulk_kind(whb_ctx *c, int kind, bool zf, dim3 grid, int off, int s, int ib, int ie, int cl, int po,
                      const StepMaps &mp) {
    if (kind == K_FIRST) {
        if (zf) launch_bulk<A1, K_FIRST, true, TENSOR>(c, grid, off, s, ib, ie, cl, po, mp);
        else launch_bulk<A1, K_FIRST, false, TENSOR>(c, grid, off, s, ib, ie, cl, po, mp);
    } else if (kind == K_MID) {
        if (zf) launch_bulk<A1, K_MID, true, TENSOR>(c, grid, off, s, ib, ie, cl, po, mp);
        else launch_bulk<A1, K_MID, false, TENSOR>(c, grid, off, s, ib, ie, cl, po, mp);
    } else {
        if (zf) launch_bulk<A1, K_LAST, true, TENSOR>(c, grid, off, s, ib, ie, cl, po, mp);
        else launch_bulk<A1, K_LAST, false, TENSOR>(c, grid, off, s, ib, ie, cl, po, mp);
    }
}

// Tensor map of one field buffer viewed as (planes, n1, pitch) float64 with a (BY+2)x(TX+4)
// box (w, with halo) or a BY x TX box (prev / f / acc).  Cached per (pointer, box).
int tensor_map(whb_ctx *c, const double *base, int box_w, int box_h, CUtensorMap *out);

// Launch step s for the first `nact` members of the table (sorted by n_total,
// descending).  The bulk kernel is specialised on the step kind, so members
// finishing at this step (LAST) get their own launch.
int launch_step_members(whb_ctx *c, int s, int moff, int nact, int i_begin, int i_end, int chunk_len, int part_off) {
    if (nact <= 0 || i_begin >= i_end) return 0;
    if (c->kern == 3) {
        if (moff != 0) return fail(WHB_E_STATE, "general kernel launches start at member 0");
        if (c->gm_nch > 0) {
            dim3 grid(c->gm_gx, c->gm_jy * c->gm_nch, nact);
            if (c->geomg.order == 4)
                step_general_march_kernel<2><<<grid, 128, 0, c->stream>>>(c->geomg, c->d_members, s, (int)c->nloc,
                                                                         c->gm_chunk, c->gm_jy);
            else
                step_general_march_kernel<1><<<grid, 128, 0, c->stream>>>(c->geomg, c->d_members, s, (int)c->nloc,
                                                                         c->gm_chunk, c->gm_jy);
        } else {
            step_general_kernel<<<dim3(kGenBlocks, nact, 1), 256, 0, c->stream>>>(c->geomg, c->d_members, s,
                                                                              (int)c->nloc, part_off);
        }
        c->launches++;
        WHB_CUDA(cudaGetLastError());
        return 0;
    }
    const int nch = (i_end - i_begin + chunk_len - 1) / chunk_len;
    if (c->kern >= 1) {
        const bool zf = c->cur_zf != 0;
        StepMaps mp;
        std::memset(&mp, 0, sizeof(mp));
        if (c->kern == 2) {
            // member 0 of the current table (nbatch == 1): buffers of this step
            const Member &m0 = c->h_members[0];
            const double *wcur = level_ptr(m0, s);
            const double *wprv = level_ptr(m0, s - 1);
            WHB_TRY(tensor_map(c, wcur, B3_TX + 4, B3_BY + 2, &mp.w));
            WHB_TRY(tensor_map(c, wprv, B3_TX, B3_BY, &mp.p));
            WHB_TRY(tensor_map(c, m0.acc, B3_TX, B3_BY, &mp.a));
            if (m0.f) WHB_TRY(tensor_map(c, m0.f, B3_TX, B3_BY, &mp.f));
        }
        int nlast = 0;
        for (int pos = moff; pos < moff + nact; ++pos) nlast += (c->mem[c->order[pos]].n_total - 1 == s);
        const int nmid = nact - nlast;
        auto go = [&](int kind, int off_rel, int cnt) {
            if (cnt <= 0) return;
            const int off = moff + off_rel;
            dim3 grid(c->gx, c->JT * nch, cnt);
            if (c->act1) {
                if (c->kern == 2) launch_bulk_kind<true, true>(c, kind, zf, grid, off, s, i_begin, i_end, chunk_len, part_off, mp);
                else launch_bulk_kind<true, false>(c, kind, zf, grid, off, s, i_begin, i_end, chunk_len, part_off, mp);
            } else
                launch_bulk_kind<false, false>(c, kind, zf, grid, off, s, i_begin, i_end, chunk_len, part_off, mp);
            c->launches++;
        };
        if (s == 0) go(K_FIRST, 0, nact);
        else {
            go(K_MID, 0, nmid);
            go(K_LAST, nmid, nlast);
        }
        WHB_CUDA(cudaGetLastError());
        return 0;
    }
    if (moff != 0) return fail(WHB_E_STATE, "simple kernel launches start at member 0");
    dim3 grid(c->gx, c->JT * nch, nact);
    dim3 block(c->BX, c->BY, 1);
    if (c->act1)
        step_kernel<true, true><<<grid, block, 0, c->stream>>>(c->geom, c->d_members, s, i_begin, i_end,
                                                             chunk_len, c->JT, part_off);
    else if (c->act0)
        step_kernel<true, false><<<grid, block, 0, c->stream>>>(c->geom, c->d_members, s, i_begin, i_end,
                                                              chunk_len, c->JT, part_off);
    else
        step_kernel<false, false><<<grid, block, 0, c->stream>>>(c->geom, c->d_members, s, i_begin, i_end,
                                                               chunk_len, c->JT, part_off);
    c->launches++;
    WHB_CUDA(cudaGetLastError());
    return 0;
}

int tensor_map(whb_ctx *c, const double *base, int box_w, int box_h, CUtensorMap *out) {
    auto key = std::make_tuple(base, box_w, box_h);
    auto it = c->tmaps.find(key);
    if (it != c->tmaps.end()) {
        *out = it->second;
        return 0;
    }
    WHB_TRY(get_encoder());
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)c->P, (cuuint64_t)c->gshape[1], (cuuint64_t)c->nplanes};
    cuuint64_t strides[2] = {(cuuint64_t)c->P * sizeof(double), (cuuint64_t)c->S0 * sizeof(double)};
    cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    // L2 promotion (the granularity a box row is fetched into L2 with): WHB_TMA_PROMO=0|64|128|256.
    // Measured on config 4 (DRAM read per three-step pass, pass time): 256 B 51.1 GB 12.92 ms, 128 B
    // 48.4 GB 12.57 ms, none 48.3 GB 12.54 ms, 64 B 46.7 GB 12.34 ms.
    static const CUtensorMapL2promotion promo = [] {
        const char *e = getenv("WHB_TMA_PROMO");
        const int v = e ? atoi(e) : 64;
        return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
             : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }();
    CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(base), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(WHB_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    c->tmaps.emplace(key, m);
    *out = m;
    return 0;
}

int launch_step(whb_ctx *c, int s, int nact, int i_begin, int i_end, int chunk_len, int part_off) {
    return launch_step_members(c, s, 0, nact, i_begin, i_end, chunk_len, part_off);
}

// one-step kernel for table members [moff, moff+cnt) over all update planes
int launch_step_range(whb_ctx *c, int s, int moff, int cnt) {
    return launch_step_members(c, s, moff, cnt, c->upd_lo, c->upd_hi, c->chunk_len, 0);
}

template <bool A1, int K1, int K2, bool ZF>
void launch_tb2(whb_ctx *c, dim3 grid, int off, int s, int ib, int ie, int cl, int po, const StepMaps &mp) {
    constexpr int threads = A1 ? T3_TX * T3_BY / 2 : T2_TX * T2_BY / 2;
    auto go = [&](auto gm) {
        tb2_fn<A1, K1, K2, ZF, decltype(gm)::value>()<<<grid, threads, c->smem2, c->stream>>>(
            c->geom, c->d_members, off, s, ib, ie, cl, (int)(grid.y / ((ie - ib + cl - 1) / cl)), po, c->win_j0,
            c->win_j1, mp.w, mp.p, mp.f, mp.a);
    };
    const int gm = geom_mode(c);
    if (gm == 2) go(std::integral_constant<int, 2>{});
    else if (gm == 1) go(std::integral_constant<int, 1>{});
    else go(std::integral_constant<int, 0>{});
}

template <bool A1>
void launch_tb2_kinds(whb_ctx *c, int k1, int k2, bool zf, dim3 grid, int off, int s, int ib, int ie, int cl,
                      int po, const StepMaps &mp) {
#define WHB_TB2_CASE(K1, K2)                                                         \
    if (k1 == K1 && k2 == K2) {                                                      \
        if (zf) launch_tb2<A1, K1, K2, true>(c, grid, off, s, ib, ie, cl, po, mp);  \
        else launch_tb2<A1, K1, K2, false>(c, grid, off, s, ib, ie, cl, po, mp);    \
        return;                                                                      \
    }
    WHB_TB2_CASE(K_FIRST, K_MID)
    WHB_TB2_CASE(K_MID, K_MID)
    WHB_TB2_CASE(K_MID, K_LAST)
    WHB_TB2_CASE(K_FIRST, K_LAST)
#undef WHB_TB2_CASE
}

// Fused steps (s, s+1) over update planes [ib, ie) in chunks of cl planes (partial slots from
// po), for the table members [0, nact): those still running after s+1 get (K1, MID), those
// finishing at s+1 get (K1, LAST).
int launch_pair_range(whb_ctx *c, int s, int ib, int ie, int cl, int po) {
    if (ib >= ie) return 0;
    const int nch = (ie - ib + cl - 1) / cl;
    int n_cont = 0, n_last = 0;
    for (int pos = 0; pos < c->nbatch; ++pos) {
        const int N = c->mem[c->order[pos]].n_total;
        n_cont += (N > s + 2);
        n_last += (N == s + 2);
    }
    if (n_cont + n_last == 0) return 0;
    const bool zf = c->cur_zf != 0;
    StepMaps mp;
    std::memset(&mp, 0, sizeof(mp));
    if (c->act1) {  // 3D: TMA tensor boxes of member 0 (nbatch == 1)
        const Member &m0 = c->h_members[0];
        WHB_TRY(tensor_map(c, level_ptr(m0, s), T3_TX + 4, T3_BY + 4, &mp.w));
        WHB_TRY(tensor_map(c, level_ptr(m0, s - 1), T3_TX + 4, T3_BY + 2, &mp.p));
        WHB_TRY(tensor_map(c, m0.acc, T3_TX, T3_BY, &mp.a));
        if (m0.f) WHB_TRY(tensor_map(c, m0.f, T3_TX + 4, T3_BY + 2, &mp.f));
    }
    const int k1 = (s == 0) ? K_FIRST : K_MID;
    auto go = [&](int k2, int off, int cnt) {
        if (cnt <= 0) return;
        int jt2 = c->JT2;
        if (c->win_j1 != INT_MAX && c->act1) {  // row window (banded host iteration)
            const int rows = std::min(c->win_j1, (int)c->gshape[1] - 1) - c->win_j0;
            jt2 = (std::max(rows, 1) + T3_BY - 1) / T3_BY;
        }
        dim3 grid(c->gx2, jt2 * nch, cnt);
        if (c->act1) launch_tb2_kinds<true>(c, k1, k2, zf, grid, off, s, ib, ie, cl, po, mp);
        else launch_tb2_kinds<false>(c, k1, k2, zf, grid, off, s, ib, ie, cl, po, mp);
        c->launches++;
    };
    go(K_MID, 0, n_cont);
    go(K_LAST, n_cont, n_last);
    WHB_CUDA(cudaGetLastError());
    return 0;
}

int launch_pair(whb_ctx *c, int s) { return launch_pair_range(c, s, c->upd_lo, c->upd_hi, c->chunk2, 0); }

// Steps (s, s+1, s+2) of the single member in one pass (step_t3.cuh); `last` when they end the solve.
int launch_t3(whb_ctx *c, int s, bool last, int ib, int ie, int cl) {
    if (ib >= ie) return 0;
    const bool zf = c->cur_zf != 0;
    const Member &m0 = c->h_members[0];
    const MemberHost &mh = c->mem[c->order[0]];
    CUtensorMap tw, tp, tf, ta, ew, ep, ef, ea;
    std::memset(&tp, 0, sizeof(tp));
    std::memset(&tf, 0, sizeof(tf));
    using SM = t3::Main;
    WHB_TRY(tensor_map(c, level_ptr(m0, s), SM::RW, SM::WR, &tw));
    WHB_TRY(tensor_map(c, level_ptr(m0, s - 1), SM::LW, SM::NR, &tp));
    if (m0.f) WHB_TRY(tensor_map(c, m0.f, SM::LW, SM::NR, &tf));
    WHB_TRY(tensor_map(c, m0.acc, SM::TX, SM::BY, &ta));
    ew = tw, ep = tp, ef = tf, ea = ta;
    const int lxe_ = (c->win_j1 != INT_MAX && c->win_lxe) ? c->win_lxe : c->lxe3;
    if (lxe_ != 32) {  // boxes of the ragged-edge shape
        const int lw = 2 * lxe_, nr = 16 * (32 / lxe_);
        WHB_TRY(tensor_map(c, level_ptr(m0, s), lw + 4, nr + 2, &ew));
        WHB_TRY(tensor_map(c, level_ptr(m0, s - 1), lw, nr, &ep));
        if (m0.f) WHB_TRY(tensor_map(c, m0.f, lw, nr, &ef));
        WHB_TRY(tensor_map(c, m0.acc, lw - 4, nr - 4, &ea));
    }
    t3::Scal sc;
    const bool first = (s == 0);
    sc.h1 = first ? mh.half_dt2 : mh.dt2;
    sc.cos1 = first ? 1.0 : mh.h_cos[s];
    sc.cos2 = mh.h_cos[s + 1];
    sc.cos3 = mh.h_cos[s + 2];
    sc.dt2 = mh.dt2;
    sc.c0 = mh.h_acc[0];
    sc.c1 = mh.h_acc[s + 1];
    sc.c2 = mh.h_acc[s + 2];
    sc.c3 = mh.h_acc[s + 3];
    sc.osc = mh.out_scale;
    const int nch = (ie - ib + cl - 1) / cl;
    // row tiles of the launch: the whole grid, or the row window [win_j0, win_j1)
    int jt = c->JT3, jte = c->JTE3;
    const int lxe = (c->win_j1 != INT_MAX && c->win_lxe) ? c->win_lxe : c->lxe3;
    if (c->win_j1 != INT_MAX) {
        const int rows = std::min(c->win_j1, (int)c->gshape[1] - 1) - c->win_j0;
        if (rows <= 0) return 0;
        const int bye = 16 * (32 / lxe) - 4;
        jt = (rows + t3::BY - 1) / t3::BY;
        jte = (rows + bye - 1) / bye;
    }
    dim3 grid(c->gx3, jt * nch, 1);
    // edge column: its jt * nch CTAs as jte row tiles x as many chunks as fit (whole grid: the same chunks)
    int cle = cl;
    if (c->win_j1 != INT_MAX && lxe != 32) {
        const int nche = std::max(1, (jt * nch) / std::max(1, jte));
        cle = std::max(1, (ie - ib + nche - 1) / nche);
    }
    int sms3 = 148;
    cudaDeviceGetAttribute(&sms3, cudaDevAttrMultiProcessorCount, c->device);
    static const char *ord = getenv("WHB_T3_ORDER");  // jt | x: force a CTA -> tile order (A/B)
    const int jt_fast = ord ? (std::string(ord) == "jt") : (c->gx3 * jt <= sms3);
    const t3::RowWin rw{c->win_j0, c->win_j1, c->win_po, jt_fast};
    const int gm = geom_mode(c);
    auto go = [&](auto k1, auto k2, auto zft, auto gmt) {
        t3_by_lxe(lxe, [&](auto lx) {
            t3_fn<decltype(k1)::value, decltype(k2)::value, decltype(zft)::value, decltype(gmt)::value,
                  decltype(lx)::value>()<<<grid, S3_THREADS, t3_smem(lxe), c->stream>>>(
                c->geom, c->d_members, s, ib, ie, cl, jt, jte, cle, rw, sc, tw, tp, tf, ta, ew, ep, ef, ea);
        });
    };
    using KF = std::integral_constant<int, K_FIRST>;
    using KM = std::integral_constant<int, K_MID>;
    using KL = std::integral_constant<int, K_LAST>;
    auto by_gm = [&](auto k1, auto k2, auto zft) {
        if (gm == 2) go(k1, k2, zft, std::integral_constant<int, 2>{});
        else if (gm == 1) go(k1, k2, zft, std::integral_constant<int, 1>{});
        else go(k1, k2, zft, std::integral_constant<int, 0>{});
    };
    auto by_zf = [&](auto k1, auto k2) {
        if (zf) by_gm(k1, k2, std::true_type{});
        else by_gm(k1, k2, std::false_type{});
    };
    if (first && last) return fail(WHB_E_STATE, "t3: a pass may not be both the first and the last");
    if (first) by_zf(KF{}, KM{});
    else if (last) by_zf(KM{}, KL{});
    else by_zf(KM{}, KM{});
    c->launches++;
    WHB_CUDA(cudaGetLastError());
    return 0;
}

int max_steps(whb_ctx *c);

template <int T, int K1, int K2, bool ZF>
void launch_wf(whb_ctx *c, int off, int cnt, int s) {
    // Row chunks per strip: one wave of CTAs for a single member (nchw); with cnt members
    // per launch, longer chunks — every chunk re-streams T + lag warm-up rows (8 at T = 4),
    // which at the single-member chunk length of a 1025^2 grid (12 rows) is 67 % extra.
    // The chunk count of a batched launch maximises (fill of the CTA waves) x (useful rows per
    // chunk): the kernel is latency-bound, so an SM holding 2 of its 3 CTAs runs at 2/3 -- 64
    // members x 5 strips as one chunk each are 320 CTAs on 444 slots (72 %), as 4 chunks each 1280
    // CTAs on 3 waves (96 %, x 256 / 264 useful rows).  WHB_WF_BATCH=wave: the old rule (one wave).
    int nch = c->nchw[T], cl = c->chw[T];
    if (cnt > 1) {
        static const bool one_wave = getenv("WHB_WF_BATCH") && std::string(getenv("WHB_WF_BATCH")) == "wave";
        const int nplanes = c->upd_hi - c->upd_lo;
        const long long res = std::max<long long>(1, c->wf_res[T]);
        int best = 1;
        if (one_wave) {
            best = (int)std::max<long long>(1, std::min<long long>(nch, res / ((long long)c->gxw[T] * cnt)));
        } else {
            double best_eff = 0.0;
            for (int n = 1; n <= c->nchw[T]; ++n) {
                const int l = (nplanes + n - 1) / n;
                const long long ctas = (long long)c->gxw[T] * ((nplanes + l - 1) / l) * cnt;
                const double eff = (double)ctas / (double)((ctas + res - 1) / res * res) * l / (l + 2.0 * T);
                if (eff > best_eff + 1e-9) best_eff = eff, best = n;
            }
        }
        cl = (nplanes + best - 1) / best;
        nch = (nplanes + cl - 1) / cl;
    }
    dim3 grid(c->gxw[T], nch, cnt);
    // per-member pass scalars (the reference's host expressions, as in the member table)
    auto fill = [&](wf2d::WfScal &ps, const MemberHost &m) {
        for (int t = 1; t <= T; ++t) {
            const bool first = (K1 == K_FIRST) && (t == 1);
            ps.h[t] = first ? m.half_dt2 : m.dt2;
            ps.cs[t] = first ? 1.0 : m.h_cos[s + t - 1];
            ps.ca[t] = m.h_acc[s + t];
        }
        ps.acc0 = m.h_acc[0];
        ps.osc = m.out_scale;
    };
    wf2d::WfTab<1> ps1{};
    wf2d::WfTab<wf2d::WF_TAB> psn;  // copied into the launch parameters at the launch
    if (cnt == 1) {
        fill(ps1.m[0], c->mem[c->order[off]]);
    } else {
        for (int z = 0; z < cnt; ++z) fill(psn.m[z], c->mem[c->order[off + z]]);
    }
    const Geom &g = c->geom;
    const int gm = geom_mode(c);
    auto go = [&](auto ps_tag, auto gm_tag) {
        constexpr bool PS = decltype(ps_tag)::value;
        auto fn = wf_fn<T, K1, K2, ZF, PS, decltype(gm_tag)::value>();
        if constexpr (PS)
            fn<<<grid, 32 * (WF_NW + 1), c->smemw[T], c->stream>>>(g, c->d_members, off, s, c->upd_lo, c->upd_hi, cl,
                                                                  0, ps1);
        else
            fn<<<grid, 32 * (WF_NW + 1), c->smemw[T], c->stream>>>(g, c->d_members, off, s, c->upd_lo, c->upd_hi, cl,
                                                                  0, psn);
    };
    using G0 = std::integral_constant<int, 0>;
    using G1 = std::integral_constant<int, 1>;
    using G2 = std::integral_constant<int, 2>;
    if (cnt == 1) {  // one member: pass scalars as kernel parameters
        if (gm == 2) go(std::true_type{}, G2{});
        else if (gm == 1) go(std::true_type{}, G1{});
        else go(std::true_type{}, G0{});
    } else {
        if (gm == 2) go(std::false_type{}, G2{});
        else if (gm == 1) go(std::false_type{}, G1{});
        else go(std::false_type{}, G0{});
    }
}

template <int T>
void launch_wf_kinds(whb_ctx *c, int k1, int k2, bool zf, int off, int cnt, int s) {
#define WHB_WF_CASE(K1, K2)                                            \
    if (k1 == K1 && k2 == K2) {                                        \
        if (zf) launch_wf<T, K1, K2, true>(c, off, cnt, s);            \
        else launch_wf<T, K1, K2, false>(c, off, cnt, s);              \
        return;                                                        \
    }
    WHB_WF_CASE(K_FIRST, K_MID)
    WHB_WF_CASE(K_MID, K_MID)
    WHB_WF_CASE(K_MID, K_LAST)
    WHB_WF_CASE(K_FIRST, K_LAST)
#undef WHB_WF_CASE
}

// One wavefront pass group: table members [off, off+cnt) advance T steps from step s.
int launch_wf_group(whb_ctx *c, int T, int off, int cnt, int s, bool last) {
    if (cnt <= 0) return 0;
    if (cnt > wf2d::WF_TAB) {  // one launch per WF_TAB members (the launch parameters hold their scalars)
        for (int o = 0; o < cnt; o += wf2d::WF_TAB)
            WHB_TRY(launch_wf_group(c, T, off + o, std::min(wf2d::WF_TAB, cnt - o), s, last));
        return 0;
    }
    const int k1 = s == 0 ? K_FIRST : K_MID;
    const int k2 = last ? K_LAST : K_MID;
    const bool zf = c->cur_zf != 0;
    if (T == 4) launch_wf_kinds<4>(c, k1, k2, zf, off, cnt, s);
    else launch_wf_kinds<2>(c, k1, k2, zf, off, cnt, s);
    c->launches++;
    WHB_CUDA(cudaGetLastError());
    return 0;
}

// Passes of wfT steps; a member with r < wfT steps left finishes with a 2-step pass and/or a
// single step.  Members are sorted by n_total (descending), so every group is contiguous.
int enqueue_wf(whb_ctx *c) {
    const int T = c->wfT;
    const int ns = max_steps(c);
    for (int s = 0; s < ns; s += T) {
        // remaining steps per table position
        int cnt_full_mid = 0, cnt_full_last = 0, cnt_r[4] = {0, 0, 0, 0};
        int pos = 0;
        for (; pos < c->nbatch; ++pos) {
            const int rem = c->mem[c->order[pos]].n_total - s;
            if (rem > T) ++cnt_full_mid;
            else if (rem == T) ++cnt_full_last;
            else if (rem > 0) ++cnt_r[rem];
        }
        int off = 0;
        WHB_TRY(launch_wf_group(c, T, off, cnt_full_mid, s, false));
        off += cnt_full_mid;
        WHB_TRY(launch_wf_group(c, T, off, cnt_full_last, s, true));
        off += cnt_full_last;
        if (T == 4) {
            // rem 3: 2-step pass (then a single last step); rem 2: 2-step last pass; rem 1: single
            WHB_TRY(launch_wf_group(c, 2, off, cnt_r[3], s, false));
            WHB_TRY(launch_wf_group(c, 2, off + cnt_r[3], cnt_r[2], s, true));
            if (cnt_r[3] > 0) WHB_TRY(launch_step_range(c, s + 2, off, cnt_r[3]));
            off += cnt_r[3] + cnt_r[2];
        }
        if (cnt_r[1] > 0) WHB_TRY(launch_step_range(c, s, off, cnt_r[1]));
    }
    return 0;
}

int max_steps(whb_ctx *c) {
    int mx = 0;
    for (auto &m : c->mem) mx = std::max(mx, m.n_total);
    return mx;
}

int active_members(whb_ctx *c, int s) {
    int n = 0;
    for (auto &m : c->mem) n += (m.n_total > s);
    return n;
}

// Shared memory of a cluster-resident launch over the current members (0: does not fit).
size_t cres_smem(whb_ctx *c) {
    if (!c->cres || c->kern == 3) return 0;
    const size_t b = cres::smem_doubles(c->cres_r, (int)c->gshape[2], max_steps(c), c->cres_cl) * sizeof(double);
    return b <= kCresSmemMax ? b : 0;
}

// One cluster per member (table positions [0, nbatch)); iters > 1 (FPI) runs that many fixed-point
// iterations inside the launch, hist == nullptr leaves the residual in partials[0] for the reduction.
int launch_cres(whb_ctx *c, size_t smem, int iters, double tol_sq, double *hist, int k0, int *done,
                double tol = -1.0, double root_n = 0.0) {
    cres::Args a{};
    a.tol = tol;
    a.root_n = root_n;
    a.CL = c->cres_cl;
    a.R = c->cres_r;
    a.W = (int)c->gshape[2];
    a.nmax = max_steps(c);
    a.iters = iters;
    a.tol_sq = tol_sq;
    a.hist = hist;
    a.k0 = k0;
    a.nb = c->nbatch;
    a.done = done;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->cres_cl, c->nbatch, 1);
    cfg.blockDim = dim3(cres::NT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c->cres_cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const Geom &g = c->geom;
    const int gm = geom_mode(c);
    const bool zf = c->cur_zf != 0;
    cudaError_t e = cudaErrorInvalidValue;
    const Member *mt = c->d_members;
#define WHB_CRES_GO(PPT)                                                                               \
    if (c->cres_ppt == PPT) {                                                                          \
        if (zf) e = gm == 2   ? cudaLaunchKernelEx(&cfg, cres_fn<true, 2, PPT>(), g, mt, 0, a)         \
                    : gm == 1 ? cudaLaunchKernelEx(&cfg, cres_fn<true, 1, PPT>(), g, mt, 0, a)         \
                              : cudaLaunchKernelEx(&cfg, cres_fn<true, 0, PPT>(), g, mt, 0, a);        \
        else e = gm == 2   ? cudaLaunchKernelEx(&cfg, cres_fn<false, 2, PPT>(), g, mt, 0, a)           \
                 : gm == 1 ? cudaLaunchKernelEx(&cfg, cres_fn<false, 1, PPT>(), g, mt, 0, a)           \
                           : cudaLaunchKernelEx(&cfg, cres_fn<false, 0, PPT>(), g, mt, 0, a);          \
    }
    WHB_CRES_GO(1) WHB_CRES_GO(2) WHB_CRES_GO(4) WHB_CRES_GO(8)
#undef WHB_CRES_GO
    WHB_CUDA(e);
    c->launches++;
    return 0;
}

// Enqueue one full filtered solve (all steps + residual reduction).
int enqueue_solve(whb_ctx *c, int out_mode) {
    const int ns = max_steps(c);
    if (const size_t cs = cres_smem(c)) {
        WHB_TRY(launch_cres(c, cs, 1, -1.0, nullptr, 0, nullptr));
        if (out_mode == WHB_OUT_FPI) {
            reduce_partials_kernel<<<1, 1024, 0, c->stream>>>(c->d_members, c->nbatch, 1, c->d_hist, c->d_counter);
            c->launches++;
            WHB_CUDA(cudaGetLastError());
        }
        return 0;
    }
    if (c->wfT) {
        WHB_TRY(enqueue_wf(c));
    } else if (c->t3 && ns > 3) {
        // passes of 3 steps; a remainder of 2 is one two-step pass, of 1 a single step
        int s = 0;
        while (ns - s >= 3) {
            WHB_TRY(launch_t3(c, s, ns - s == 3, c->upd_lo, c->upd_hi, c->chunk3));
            s += 3;
        }
        if (ns - s == 2) WHB_TRY(launch_pair(c, s));
        else if (ns - s == 1) WHB_TRY(launch_step_range(c, s, 0, 1));
    } else if (c->tb2) {
        // pairs (0,1), (2,3), ...; a member with odd n_total takes its last step alone
        for (int s = 0; s < ns; s += 2) {
            WHB_TRY(launch_pair(c, s));
            int n_single = 0, off = 0;
            for (int pos = 0; pos < c->nbatch; ++pos) {
                const int N = c->mem[c->order[pos]].n_total;
                if (N > s + 1) ++off;
                n_single += (N == s + 1);
            }
            if (n_single > 0) WHB_TRY(launch_step_range(c, s, off, n_single));
        }
    } else {
        for (int s = 0; s < ns; ++s)
            WHB_TRY(launch_step(c, s, active_members(c, s), c->upd_lo, c->upd_hi, c->chunk_len, 0));
    }
    if (out_mode == WHB_OUT_FPI) {
        int np = c->kern == 3 ? (c->gm_nch > 0 ? c->gm_gx * c->gm_jy * c->gm_nch : kGenBlocks)
                              : c->gx * c->JT * c->nchunks;
        if (c->tb2) np = std::max(np, c->gx2 * c->JT2 * c->nch2);
        if (c->t3) np = std::max(np, c->gx3 * c->JT3 * c->nch3);
        if (c->wfT) np = std::max(np, std::max(c->gxw[2] * c->nchw[2], c->wfT == 4 ? c->gxw[4] * c->nchw[4] : 0));
        reduce_partials_kernel<<<1, 1024, 0, c->stream>>>(c->d_members, c->nbatch, np, c->d_hist, c->d_counter);
        c->launches++;
        WHB_CUDA(cudaGetLastError());
    }
    return 0;
}

int run_solve(whb_ctx *c, int out_mode, int zf) {
    c->cur_zf = zf;  // the bulk kernel is specialised on zero forcing
    if (!c->use_graphs) return enqueue_solve(c, out_mode);
    // the 3D TMA path bakes member 0's tensor maps (its v buffer) into the graph
    const void *vkey = (c->kern == 2 && !c->h_members.empty()) ? (const void *)c->h_members[0].v : nullptr;
    auto key = std::make_tuple(out_mode, zf, vkey);
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
        cudaGraph_t g;
        const int64_t l0 = c->launches;
        WHB_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_solve(c, out_mode);
        cudaError_t e = cudaStreamEndCapture(c->stream, &g);
        if (rc) return rc;
        if (e != cudaSuccess) return fail(WHB_E_CUDA, std::string("capture: ") + cudaGetErrorString(e));
        cudaGraphExec_t ge;
        e = cudaGraphInstantiate(&ge, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return fail(WHB_E_CUDA, std::string("instantiate: ") + cudaGetErrorString(e));
        c->graph_kernels[key] = c->launches - l0;
        c->launches = l0;
        it = c->graphs.emplace(key, ge).first;
    }
    WHB_CUDA(cudaGraphLaunch(it->second, c->stream));
    c->launches += c->graph_kernels[key];  // kernels the graph launches
    return 0;
}

int ensure_events(whb_ctx *c, int n) {
    while ((int)c->ev.size() < n) {
        cudaEvent_t e;
        WHB_CUDA(cudaEventCreate(&e));
        c->ev.push_back(e);
    }
    return 0;
}

int check_ready(whb_ctx *c) {
    if (!c->op_set) return fail(WHB_E_STATE, "operator not set (whb_set_operator)");
    for (int b = 0; b < c->nbatch; ++b)
        if (c->mem[b].n_total < 2) return fail(WHB_E_STATE, "schedule not set for member " + std::to_string(b));
    return 0;
}

// Stopping test of the fixed-point loop for one member's resid^2: root_n > 0 follows
// driver.py:225-230 exactly (sqrt(r) / sqrt(N) <= tol, IEEE sqrt and division), else r <= tol_sq.
bool fpi_stop(double r, double tol_sq, double tol, double root_n) {
    if (root_n > 0.0) return tol >= 0.0 && std::sqrt(r) / root_n <= tol;
    return tol_sq >= 0.0 && r <= tol_sq;
}

int fpi_impl(whb_ctx *c, int iters, double tol_sq, double *resid_out, int *done, double tol = -1.0,
             double root_n = 0.0) {
    const bool checks = root_n > 0.0 ? tol >= 0.0 : tol_sq >= 0.0;
    WHB_TRY(check_ready(c));
    WHB_TRY(ensure_hist(c, iters));
    WHB_TRY(upload_members(c, WHB_OUT_FPI, 0));
    WHB_CUDA(cudaMemsetAsync(c->d_counter, 0, sizeof(int), c->stream));
    if (c->timing) WHB_TRY(ensure_events(c, 2 * iters + 2));
    int k = 0;
    std::vector<double> h(c->nbatch);
    int64_t step_kernels = 0;
    // cluster-resident grids: the whole fixed-point loop is one launch (the convergence test runs
    // in the kernel; with several members only a fixed iteration count, as the host loop stops on
    // all members together)
    c->cur_zf = 0;
    const size_t cs = cres_smem(c);
    if (cs && iters > 0 && (c->nbatch == 1 || !checks)) {
        if (c->flush_buf) {
            l2_flush_kernel<<<1184, 256, 0, c->stream>>>(c->flush_buf, c->flush_elems, 0.0);
            c->launches++;
            WHB_CUDA(cudaGetLastError());
        }
        if (c->timing) WHB_CUDA(cudaEventRecord(c->ev[0], c->stream));
        WHB_TRY(launch_cres(c, cs, iters, tol_sq, c->d_hist, 0, c->d_counter, tol, root_n));
        if (c->timing) WHB_CUDA(cudaEventRecord(c->ev[1], c->stream));
        int kd = 0;
        WHB_CUDA(cudaMemcpyAsync(&kd, c->d_counter, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        WHB_CUDA(cudaStreamSynchronize(c->stream));
        k = kd;
        if (resid_out && k > 0)
            WHB_CUDA(cudaMemcpyAsync(resid_out, c->d_hist, (size_t)k * c->nbatch * sizeof(double),
                                     cudaMemcpyDeviceToHost, c->stream));
        WHB_CUDA(cudaStreamSynchronize(c->stream));
        if (c->timing) {
            float ms = 0.f;
            WHB_CUDA(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
            c->t_solve_ms = ms;
            c->t_step_ms = ms;
            c->t_step_launches = 1;
        }
        if (done) *done = k;
        return 0;
    }
    for (k = 0; k < iters; ++k) {
        if (c->flush_buf) {
            l2_flush_kernel<<<1184, 256, 0, c->stream>>>(c->flush_buf, c->flush_elems, (double)k);
            c->launches++;
            WHB_CUDA(cudaGetLastError());
        }
        if (c->timing) WHB_CUDA(cudaEventRecord(c->ev[2 * k], c->stream));
        const int64_t l0 = c->launches;
        WHB_TRY(run_solve(c, WHB_OUT_FPI, 0));
        step_kernels += c->launches - l0 - 1;  // minus the residual reduction
        if (c->timing) WHB_CUDA(cudaEventRecord(c->ev[2 * k + 1], c->stream));
        if (checks) {
            WHB_CUDA(cudaMemcpyAsync(h.data(), c->d_hist + (size_t)k * c->nbatch, c->nbatch * sizeof(double),
                                     cudaMemcpyDeviceToHost, c->stream));
            WHB_CUDA(cudaStreamSynchronize(c->stream));
            bool conv = true;
            for (double r : h) conv = conv && fpi_stop(r, tol_sq, tol, root_n);
            if (conv) {
                ++k;
                break;
            }
        }
    }
    if (resid_out && k > 0)
        WHB_CUDA(cudaMemcpyAsync(resid_out, c->d_hist, (size_t)k * c->nbatch * sizeof(double),
                                 cudaMemcpyDeviceToHost, c->stream));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    if (c->timing) {
        double tot = 0.0;
        for (int i = 0; i < k; ++i) {
            float ms = 0.f;
            WHB_CUDA(cudaEventElapsedTime(&ms, c->ev[2 * i], c->ev[2 * i + 1]));
            tot += ms;
        }
        c->t_solve_ms = tot;
        c->t_step_ms = tot;
        c->t_step_launches = step_kernels;
    }
    if (done) *done = k;
    return 0;
}

// Host <-> device field copies.  The device rows are pitched; a 2D copy engine
// transfer of n2-element rows can be slower than one contiguous transfer, so by
// default the host data moves contiguously into a staging buffer and a kernel
// scatters it into the pitched layout (and the reverse for downloads).
// WHB_STAGED=0 uses cudaMemcpy2DAsync directly.
int ensure_stage(whb_ctx *c) {
    if (c->stage) return 0;
    const size_t n = (size_t)c->nloc * c->gshape[1] * c->gshape[2];
    WHB_CUDA(cudaMalloc(&c->stage, n * sizeof(double)));
    return 0;
}

bool staged(whb_ctx *c) {
    static const char *e = getenv("WHB_STAGED");
    return !(e && std::string(e) == "0") && c->P != c->gshape[2];
}

int copy_field_h2d(whb_ctx *c, double *dev, const double *host) {
    // host: owned planes C-contiguous (nloc, n1, n2); device rows have pitch P
    const size_t rows = (size_t)c->nloc * c->gshape[1];
    if (staged(c)) {
        WHB_TRY(ensure_stage(c));
        WHB_CUDA(cudaMemcpyAsync(c->stage, host, rows * c->gshape[2] * sizeof(double), cudaMemcpyHostToDevice,
                                 c->stream));
        repitch_kernel<<<1184, 256, 0, c->stream>>>(c->stage, (int)c->gshape[2], owned(dev, c), c->P,
                                                    (long long)rows, 1);
        c->launches++;
        WHB_CUDA(cudaGetLastError());
        return 0;
    }
    WHB_CUDA(cudaMemcpy2DAsync(owned(dev, c), (size_t)c->P * sizeof(double), host,
                               (size_t)c->gshape[2] * sizeof(double), (size_t)c->gshape[2] * sizeof(double),
                               rows, cudaMemcpyHostToDevice, c->stream));
    return 0;
}

int copy_field_d2h(whb_ctx *c, const double *dev, double *host) {
    const size_t rows = (size_t)c->nloc * c->gshape[1];
    if (staged(c)) {
        WHB_TRY(ensure_stage(c));
        repitch_kernel<<<1184, 256, 0, c->stream>>>(c->stage, (int)c->gshape[2], owned(const_cast<double *>(dev), c),
                                                    c->P, (long long)rows, 0);
        c->launches++;
        WHB_CUDA(cudaGetLastError());
        WHB_CUDA(cudaMemcpyAsync(host, c->stage, rows * c->gshape[2] * sizeof(double), cudaMemcpyDeviceToHost,
                                 c->stream));
        return 0;
    }
    WHB_CUDA(cudaMemcpy2DAsync(host, (size_t)c->gshape[2] * sizeof(double), owned(dev, c),
                               (size_t)c->P * sizeof(double), (size_t)c->gshape[2] * sizeof(double), rows,
                               cudaMemcpyDeviceToHost, c->stream));
    return 0;
}

int zero_bnd(whb_ctx *c, double *x) {
    const bool gen = c->kern == 3;
    const int per0 = gen ? c->geomg.per[0] : 0;
    const int zlo = (c->act0 && !per0 && c->plane_begin == 0) ? 1 : 0;
    const int zhi = (c->act0 && !per0 && c->plane_end == c->gshape[0]) ? 1 : 0;
    zero_boundary_kernel<<<592, 256, 0, c->stream>>>(x, c->S0, c->P, (int)c->gshape[1], (int)c->gshape[2],
                                                     c->act1, GH, (int)c->nloc + GH, zlo, zhi,
                                                     gen ? c->geomg.per[1] : 0, gen ? c->geomg.per[2] : 0);
    c->launches++;
    WHB_CUDA(cudaGetLastError());
    return 0;
}

// ---- implicit-mode helpers (implicit.cuh) ---------------------------------------------------

void free_mg(whb_ctx *c) {
    if (!c->mg) return;
    for (auto &kv : c->mg->graphs) cudaGraphExecDestroy(kv.second);
    for (auto &L : c->mg->lv)
        for (double *p : L.raw)
            if (p) cudaFree(p);
    cudaFree(c->mg->ainv);
    delete c->mg;
    c->mg = nullptr;
}

void free_tri(whb_ctx *c) {
    if (!c->tri) return;
    cudaFree(c->tri->sub); cudaFree(c->tri->dp); cudaFree(c->tri->cp); cudaFree(c->tri->y);
    delete c->tri;
    c->tri = nullptr;
}

// one V-cycle from u = 0 on level `l` (linalg.py:322-339); u of the coarsest level is the
// coarse solve of b
int mg_enqueue(whb_ctx *c, int l) {
    MGData &M = *c->mg;
    MGLevelBuf &B = M.lv[l];
    const imp::Lev &L = B.lev;
    if (l == M.lc) {  // the rest of the cycle in one thread block (implicit.cuh)
        imp::coarse_cycle_kernel<<<1, 1024, M.cc_smem, c->stream>>>(M.cc, B.b, B.u, M.ainv);
        c->launches++;
        WHB_CUDA(cudaGetLastError());
        return 0;
    }
    if (l == (int)M.lv.size() - 1) {
        const int n = (L.nx - 1) * (L.ny - 1);
        imp::coarse_solve_kernel<<<std::max(1, std::min(592, (n + 7) / 8)), 256, 0, c->stream>>>(L, M.ainv, B.b, B.u);
        c->launches++;
        WHB_CUDA(cudaGetLastError());
        return 0;
    }
    // The level's current iterate: the blocked smoother cannot update in place (neighbouring CTAs
    // read their halos while it writes), so it ping-pongs between u and r (r is otherwise free:
    // the residual is formed inside the restriction); the cycle ends with the iterate in u.
    double *cur = B.u;
    auto gs = [&](int color) {
        imp::gs_color_kernel<<<std::max(1, L.nx - 1), 256, 0, c->stream>>>(L, cur, B.b, color);
        c->launches++;
    };
    // nu sweeps = 2 nu half-sweeps; with nu = 2 they run as one temporally blocked launch
    const char *gsenv = getenv("WHB_GS_BLOCK");
    const bool block4 = !(gsenv && std::string(gsenv) == "0");
    // 32 x 64 tiles while they fill the GPU, 16 x 32 on smaller levels (latency-bound there)
    const bool big = (long long)((L.ny + 63) / 64) * ((L.nx + 31) / 32) >= 4 * 148;
    auto gsb = [&](const double *uin, double *uout, int c0) {
        if (big)
            imp::gs_block_kernel<32, 64, 4><<<dim3((L.ny + 63) / 64, (L.nx + 31) / 32), 256, 0, c->stream>>>(
                L, uin, uout, B.b, c0);
        else
            imp::gs_block_kernel<16, 32, 4><<<dim3((L.ny + 31) / 32, (L.nx + 15) / 16), 256, 0, c->stream>>>(
                L, uin, uout, B.b, c0);
        c->launches++;
    };
    if (block4 && M.nu1 == 2) {
        gsb(B.u, B.r, 0);
        cur = B.r;
    } else
        for (int k = 0; k < M.nu1; ++k) { gs(0); gs(1); }
    // r = b - A u, restricted onto the next level, whose iterate starts at 0 (linalg.py:333-335)
    MGLevelBuf &N = M.lv[l + 1];
    imp::resid_restrict_kernel<<<N.lev.nx + 1, 128, 0, c->stream>>>(L, cur, B.b, N.lev, N.b, N.u);
    c->launches++;
    WHB_TRY(mg_enqueue(c, l + 1));
    imp::prolong_add_kernel<<<L.nx + 1, 256, 0, c->stream>>>(L, cur, N.lev, N.u);
    c->launches++;
    if (block4 && M.nu2 == 2 && cur != B.u) {
        gsb(cur, B.u, 1);
    } else {
        if (cur != B.u) {
            WHB_CUDA(cudaMemcpyAsync(B.u, cur, (size_t)(L.nx + 1) * L.rs * sizeof(double), cudaMemcpyDeviceToDevice,
                                     c->stream));
            cur = B.u;
        }
        for (int k = 0; k < M.nu2; ++k) { gs(1); gs(0); }
    }
    WHB_CUDA(cudaGetLastError());
    return 0;
}

// dot(x, y) over owned points into the device CG scalars (imp::cg_final_kernel mode)
int cg_dot(whb_ctx *c, const double *x, const double *y, int mode) {
    dot_partials_kernel<<<kRedBlocks, kRedThreads, 0, c->stream>>>(owned(x, c), owned(y, c), owned_elems(c), c->d_red);
    imp::cg_final_kernel<<<1, 1024, 0, c->stream>>>(c->d_red, kRedBlocks, c->d_cg, mode);
    c->launches += 2;
    WHB_CUDA(cudaGetLastError());
    return 0;
}

int imp_apply_enqueue(whb_ctx *c, const double *x, double *y, double s, double *t) {
    if (c->kern == 3) {
        apply_general_kernel<<<kGenBlocks, 256, 0, c->stream>>>(c->geomg, x, t, (int)c->nloc);
        imp::sub_scaled_kernel<<<kRedBlocks, kRedThreads, 0, c->stream>>>(owned(x, c), s, owned(t, c), owned(y, c),
                                                                           owned_elems(c));
        c->launches += 2;
    } else {
        auto kfn = c->act1 ? imp::apply_kernel<true, true>
                           : (c->act0 ? imp::apply_kernel<true, false> : imp::apply_kernel<false, false>);
        const long long rows = (long long)c->nloc * c->gshape[1];
        kfn<<<(int)std::min<long long>(rows, 1 << 20), 256, 0, c->stream>>>(c->geom, x, y, s, GH, GH + (int)c->nloc,
                                                                          c->upd_lo, c->upd_hi);
        c->launches++;
    }
    WHB_CUDA(cudaGetLastError());
    return 0;
}

// z = M r: 0 none (z is r), 1 multigrid V-cycle, 2 tridiagonal elimination
int precond_enqueue(whb_ctx *c, const double *r, double *z, int precond) {
    if (precond == 1) {
        MGData &M = *c->mg;
        M.lv[0].b = const_cast<double *>(owned(r, c));
        M.lv[0].u = owned(z, c);
        WHB_CUDA(cudaMemsetAsync(z - c->slack_front, 0,
                                 (size_t)(c->slack_front + c->field_elems + c->slack_back) * sizeof(double), c->stream));
        return mg_enqueue(c, 0);
    }
    if (precond == 2) {
        TriData &T = *c->tri;
        WHB_CUDA(cudaMemsetAsync(owned(z, c), 0, (size_t)owned_elems(c) * sizeof(double), c->stream));
        imp::tri_solve_kernel<<<1, 32, 0, c->stream>>>(owned(r, c) + 1, owned(z, c) + 1, T.n, T.sub, T.dp, T.cp, T.y);
        c->launches++;
        WHB_CUDA(cudaGetLastError());
    }
    return 0;
}

int vec_reduce_dot(whb_ctx *c, const double *x, const double *y, double *out) {
    dot_partials_kernel<<<kRedBlocks, kRedThreads, 0, c->stream>>>(owned(x, c), owned(y, c), owned_elems(c), c->d_red);
    final_sum_kernel<<<1, 1024, 0, c->stream>>>(c->d_red, kRedBlocks, c->d_red + kRedBlocks);
    c->launches += 2;
    WHB_CUDA(cudaGetLastError());
    WHB_CUDA(cudaMemcpyAsync(c->h_red, c->d_red + kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    *out = *c->h_red;
    return 0;
}

}  // namespace

// ==========================================================================================
// C ABI

// ---- NCCL (dlopen'ed: the process's already-loaded libnccl, e.g. torch's, is reused) ----------
namespace {
struct NcclApi {
    void *h = nullptr;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) err = nullptr;
} g_nccl;

int nccl_load() {
    if (g_nccl.h) return 0;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return fail(WHB_E_STATE, std::string("libnccl.so.2 not loadable: ") + dlerror());
    auto sym = [&](const char *n) { return dlsym(h, n); };
#define WHB_NCCL_SYM(field, name)                                                         \
    g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(sym(name));                  \
    if (!g_nccl.field) return fail(WHB_E_STATE, std::string("libnccl lacks ") + name);
    WHB_NCCL_SYM(get_unique_id, "ncclGetUniqueId")
    WHB_NCCL_SYM(init_rank, "ncclCommInitRank")
    WHB_NCCL_SYM(destroy, "ncclCommDestroy")
    WHB_NCCL_SYM(send, "ncclSend")
    WHB_NCCL_SYM(recv, "ncclRecv")
    WHB_NCCL_SYM(group_start, "ncclGroupStart")
    WHB_NCCL_SYM(group_end, "ncclGroupEnd")
    WHB_NCCL_SYM(all_reduce, "ncclAllReduce")
    WHB_NCCL_SYM(err, "ncclGetErrorString")
#undef WHB_NCCL_SYM
    g_nccl.h = h;
    return 0;
}

void nccl_comm_destroy(ncclComm_t comm) {
    if (comm && g_nccl.destroy) g_nccl.destroy(comm);
}

#define WHB_NCCL(call)                                                                         \
    do {                                                                                       \
        ncclResult_t _r = (call);                                                              \
        if (_r != ncclSuccess) return fail(WHB_E_CUDA, std::string(#call) + ": " + g_nccl.err(_r)); \
    } while (0)
}  // namespace

extern "C" {

int whb_abi_version(void) { return WHB_ABI_VERSION; }

const char *whb_last_error(void) { return g_last_error.c_str(); }

int whb_device_count(int *count) {
    if (!count) return fail(WHB_E_ARG, "count is NULL");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        *count = 0;
        return fail(WHB_E_NODEV, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    }
    *count = n;
    return 0;
}

int whb_create(whb_ctx **out, int device, int ndim, const int64_t *shape, int64_t plane_begin,
               int64_t plane_end, int nbatch, int shared_forcing) {
    if (!out || !shape) return fail(WHB_E_ARG, "NULL argument");
    *out = nullptr;
    if (ndim < 1 || ndim > 3) return fail(WHB_E_ARG, "ndim must be 1, 2 or 3");
    for (int a = 0; a < ndim; ++a)
        if (shape[a] < 3) return fail(WHB_E_ARG, "every axis needs at least 3 stored points");
    if (nbatch < 1) return fail(WHB_E_ARG, "nbatch must be >= 1");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(WHB_E_NODEV, "no CUDA device");
    if (device < 0 || device >= ndev) return fail(WHB_E_ARG, "device index out of range");
    whb_ctx *c = new whb_ctx();
    c->device = device;
    c->ndim = ndim;
    if (ndim == 3) {
        c->gshape[0] = shape[0]; c->gshape[1] = shape[1]; c->gshape[2] = shape[2];
        c->act0 = 1; c->act1 = 1;
    } else if (ndim == 2) {
        c->gshape[0] = shape[0]; c->gshape[1] = 1; c->gshape[2] = shape[1];
        c->act0 = 1; c->act1 = 0;
    } else {
        c->gshape[0] = 1; c->gshape[1] = 1; c->gshape[2] = shape[0];
        c->act0 = 0; c->act1 = 0;
    }
    if (ndim == 1) {
        plane_begin = 0;
        plane_end = 1;
    }
    if (plane_begin < 0 || plane_end > c->gshape[0] || plane_begin >= plane_end) {
        delete c;
        return fail(WHB_E_ARG, "invalid owned plane range");
    }
    if ((c->gshape[2] > (1 << 30)) || (c->gshape[1] > (1 << 30))) {
        delete c;
        return fail(WHB_E_ARG, "axis too large");
    }
    c->plane_begin = plane_begin;
    c->plane_end = plane_end;
    c->nloc = plane_end - plane_begin;
    c->nplanes = c->nloc + 2 * GH;
    c->P = (int)((c->gshape[2] + 15) / 16 * 16);
    c->S0 = (int64_t)c->P * c->gshape[1];
    c->field_elems = c->nplanes * c->S0;
    c->nbatch = nbatch;
    c->shared_f = shared_forcing ? 1 : 0;
    c->mem.resize(nbatch);
    c->order.resize(nbatch);
    for (int b = 0; b < nbatch; ++b) c->order[b] = b;
    const char *g = getenv("WHB_NO_GRAPHS");
    if (g && atoi(g)) c->use_graphs = false;

    auto cleanup = [&](int rc) {
        whb_destroy(c);
        return rc;
    };
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cleanup(fail(WHB_E_CUDA, cudaGetErrorString(e)));
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cleanup(fail(WHB_E_CUDA, cudaGetErrorString(e)));
    int rc = plan_launch(c);
    if (rc) return cleanup(rc);
    for (int b = 0; b < nbatch; ++b) {
        MemberHost &m = c->mem[b];
        for (int q = 0; q < c->nring && !rc; ++q) rc = alloc_field(c, &m.ring[q]);
        if (rc) return cleanup(rc);
        if ((rc = alloc_field(c, &m.v)) ||
            (rc = alloc_field(c, &m.acc)))
            return cleanup(rc);
        if (!c->shared_f && (rc = alloc_field(c, &m.f))) return cleanup(rc);
        e = cudaMalloc(&m.partials, (size_t)c->nparts * sizeof(double));
        if (e != cudaSuccess) return cleanup(fail(WHB_E_NOMEM, "partials"));
        cudaMemsetAsync(m.partials, 0, (size_t)c->nparts * sizeof(double), c->stream);
    }
    if (c->shared_f && (rc = alloc_field(c, &c->shared_f_ptr))) return cleanup(rc);
    if (cudaMalloc(&c->d_members, nbatch * sizeof(Member)) != cudaSuccess ||
        cudaMalloc(&c->d_counter, sizeof(int)) != cudaSuccess ||
        cudaMalloc(&c->d_red, (kRedBlocks + 8) * sizeof(double)) != cudaSuccess ||
        cudaMallocHost(&c->h_red, 8 * sizeof(double)) != cudaSuccess)
        return cleanup(fail(WHB_E_NOMEM, "context scratch"));
    if ((rc = ensure_hist(c, 64))) return cleanup(rc);
    e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return cleanup(fail(WHB_E_CUDA, cudaGetErrorString(e)));
    *out = c;
    return 0;
}

int whb_destroy(whb_ctx *c) {
    if (!c) return 0;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    free_mg(c);
    free_tri(c);
    drop_cg_graphs(c);
    cudaFree(c->d_cg);
    for (auto &kv : c->graphs) cudaGraphExecDestroy(kv.second);
    invalidate_user_graphs(c);
    for (auto &m : c->mem) {
        free_field(c, m.v); free_field(c, m.f); free_field(c, m.acc);
        for (int q = 0; q < 6; ++q) free_field(c, m.ring[q]);
        free_field(c, m.out);
        cudaFree(m.cos_f); cudaFree(m.acc_c); cudaFree(m.partials);
    }
    free_field(c, c->shared_f_ptr);
    for (double *v : c->vecs) free_field(c, v);
    cudaFree(c->d_members);
    cudaFree(c->d_hist);
    cudaFree(c->d_counter);
    cudaFree(c->d_red);
    cudaFree(c->flush_buf);
    cudaFree(c->stage);
    if (c->h_red) cudaFreeHost(c->h_red);
    cudaFree(c->d_mgs);
    if (c->h_mgs) cudaFreeHost(c->h_mgs);
    for (auto e : c->ev) cudaEventDestroy(e);
    for (auto e : c->ev_band) cudaEventDestroy(e);
    if (c->s_in) cudaStreamDestroy(c->s_in);
    if (c->s_out) cudaStreamDestroy(c->s_out);
    for (auto st : c->s_band) cudaStreamDestroy(st);
    if (c->nccl) nccl_comm_destroy(c->nccl);
    cudaFree(c->d_nccl);
    if (c->comm) {
        cudaStreamSynchronize(c->comm);
        cudaStreamDestroy(c->comm);
        cudaEventDestroy(c->ev_fork);
        cudaEventDestroy(c->ev_join);
    }
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return 0;
}

int whb_set_operator(whb_ctx *c, const double *clo, const double *cmid, double c2) {
    if (!c || !clo || !cmid) return fail(WHB_E_ARG, "NULL argument");
    Geom &g = c->geom;
    g.S0 = c->S0;
    g.P = c->P;
    g.n1 = (int)c->gshape[1];
    g.n2 = (int)c->gshape[2];
    g.j_lo = c->act1 ? 1 : 0;
    g.j_hi = c->act1 ? (int)c->gshape[1] - 1 : 1;
    // global-interior planes [1, n0-1) in local indices, clipped to the allocation: the two-step
    // pass of a slab computes W^{s+1} on one ghost plane per side (zero where it is global boundary)
    if (c->act0) {
        g.i_lo = (int)std::max<int64_t>(0, 1 - c->plane_begin + GH);
        g.i_hi = (int)std::min<int64_t>(c->nplanes, c->gshape[0] - 1 - c->plane_begin + GH);
    } else {
        g.i_lo = c->upd_lo;
        g.i_hi = c->upd_hi;
    }
    g.c2 = c2;
    g.use_c2 = (c2 != 1.0);  // x*1.0 == x exactly: skipping keeps bitwise parity
    // map reference axes onto storage axes: 3D (0,1,2); 2D (0,-,2); 1D (-,-,2)
    g.clo0 = g.cmid0 = g.clo1 = g.cmid1 = 0.0;
    if (c->ndim == 3) {
        g.clo0 = clo[0]; g.cmid0 = cmid[0];
        g.clo1 = clo[1]; g.cmid1 = cmid[1];
        g.clo2 = clo[2]; g.cmid2 = cmid[2];
    } else if (c->ndim == 2) {
        g.clo0 = clo[0]; g.cmid0 = cmid[0];
        g.clo2 = clo[1]; g.cmid2 = cmid[1];
    } else {
        g.clo2 = clo[0]; g.cmid2 = cmid[0];
    }
    c->op_set = true;
    return 0;
}

int whb_set_operator_general(whb_ctx *c, int order, const int *periodic, const double *taps, double c2) {
    if (!c || !periodic || !taps) return fail(WHB_E_ARG, "NULL argument");
    if (order != 2 && order != 4) return fail(WHB_E_ARG, "order must be 2 or 4");
    if (c->plane_begin != 0 || c->plane_end != (c->ndim == 1 ? 1 : c->gshape[0]))
        return fail(WHB_E_ARG, "the general operator needs a whole-grid context (no slabs)");
    WHB_TRY(set_dev(c));
    GeomG &g = c->geomg;
    std::memset(&g, 0, sizeof(g));
    g.S0 = c->S0;
    g.P = c->P;
    g.order = order;
    g.c2 = c2;
    g.use_c2 = (c2 != 1.0);
    g.plane_begin = (int)c->plane_begin;
    const int off = 3 - c->ndim;  // reference axis a -> storage axis: 3D a, 2D (0, 2), 1D 2
    for (int a = 0; a < c->ndim; ++a) {
        const int sa = (c->ndim == 2 && a == 1) ? 2 : (c->ndim == 2 ? 0 : off + a);
        g.act[sa] = 1;
        g.per[sa] = periodic[a] ? 1 : 0;
        for (int q = 0; q <= order; ++q) g.taps[sa][q] = taps[a * (order + 1) + q];
    }
    g.n[0] = (int)c->gshape[0];
    g.n[1] = (int)c->gshape[1];
    g.n[2] = (int)c->gshape[2];
    for (int a = 0; a < 3; ++a)
        if (g.act[a] && g.n[a] < order + 1) return fail(WHB_E_ARG, "axis too short for the stencil");
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    c->kern = 3;
    c->cres = false;
    c->tb2 = false;
    c->wfT = 0;
    // marching plan (WHB_GEN_MARCH=0: the grid-stride kernel): 128 columns per CTA along axis 2,
    // one CTA row per axis-1 index, axis-0 chunks so that ~4 waves of 16 CTAs per SM exist
    {
        const char *ge = getenv("WHB_GEN_MARCH");
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
        c->gm_gx = (int)((c->gshape[2] + 127) / 128);
        c->gm_jy = g.act[1] ? (int)c->gshape[1] : 1;
        const long long cols = (long long)c->gm_gx * c->gm_jy;
        const int nl = (int)c->nloc;
        long long nch = std::max<long long>(1, (4LL * sms * 16 + cols - 1) / cols);
        nch = std::min<long long>(nch, std::max(1, nl / 8));  // chunks of >= 8 planes
        c->gm_chunk = (int)((nl + nch - 1) / nch);
        if (const char *gc = getenv("WHB_GM_CHUNK")) c->gm_chunk = std::max(1, atoi(gc));
        c->gm_nch = (nl + c->gm_chunk - 1) / c->gm_chunk;
        if ((ge && std::string(ge) == "0") || (long long)c->gm_jy * c->gm_nch > 65535) c->gm_nch = 0;
    }
    for (auto &kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
    c->graph_kernels.clear();
    const int np_gen = std::max(kGenBlocks, c->gm_gx * c->gm_jy * c->gm_nch);
    if (c->nparts < np_gen) {
        c->nparts = np_gen;
        for (auto &m : c->mem) {
            cudaFree(m.partials);
            WHB_CUDA(cudaMalloc(&m.partials, (size_t)c->nparts * sizeof(double)));
            WHB_CUDA(cudaMemset(m.partials, 0, (size_t)c->nparts * sizeof(double)));
        }
        c->h_members.clear();
    }
    c->op_set = true;
    return 0;
}

int whb_set_schedule(whb_ctx *c, int member, int n_total, double half_dt2, double dt2, const double *cos_f,
                     const double *acc_c, double out_scale) {
    if (!c || !cos_f || !acc_c) return fail(WHB_E_ARG, "NULL argument");
    if (member < 0 || member >= c->nbatch) return fail(WHB_E_ARG, "member out of range");
    if (n_total < 2) return fail(WHB_E_ARG, "n_total must be >= 2");
    WHB_TRY(set_dev(c));
    MemberHost &m = c->mem[member];
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    if (m.n_total != n_total) {
        cudaFree(m.cos_f);
        cudaFree(m.acc_c);
        m.cos_f = m.acc_c = nullptr;
        WHB_CUDA(cudaMalloc(&m.cos_f, n_total * sizeof(double)));
        WHB_CUDA(cudaMalloc(&m.acc_c, (n_total + 1) * sizeof(double)));
    }
    WHB_CUDA(cudaMemcpy(m.cos_f, cos_f, n_total * sizeof(double), cudaMemcpyHostToDevice));
    WHB_CUDA(cudaMemcpy(m.acc_c, acc_c, (n_total + 1) * sizeof(double), cudaMemcpyHostToDevice));
    m.h_cos.assign(cos_f, cos_f + n_total);
    m.h_acc.assign(acc_c, acc_c + n_total + 1);
    m.n_total = n_total;
    m.half_dt2 = half_dt2;
    m.dt2 = dt2;
    m.out_scale = out_scale;
    // table order: members by n_total descending (active members form a prefix at every step)
    std::stable_sort(c->order.begin(), c->order.end(),
                     [&](int a, int b) { return c->mem[a].n_total > c->mem[b].n_total; });
    for (auto &kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
    invalidate_user_graphs(c);  // they bake the step count and the cos_f / acc_c buffers
    c->h_members.clear();
    return 0;
}

int whb_upload(whb_ctx *c, int field, int member, const double *host) {
    if (!c || !host) return fail(WHB_E_ARG, "NULL argument");
    if (member < 0 || member >= c->nbatch || field < 0 || field > WHB_WD) return fail(WHB_E_ARG, "bad field/member");
    WHB_TRY(set_dev(c));
    if (field == WHB_OUT) WHB_TRY(ensure_out(c, member));
    double *d = field_ptr(c, field, member);
    WHB_TRY(copy_field_h2d(c, d, host));
    WHB_TRY(zero_bnd(c, d));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
}

int whb_download(whb_ctx *c, int field, int member, double *host) {
    if (!c || !host) return fail(WHB_E_ARG, "NULL argument");
    if (member < 0 || member >= c->nbatch || field < 0 || field > WHB_WD) return fail(WHB_E_ARG, "bad field/member");
    WHB_TRY(set_dev(c));
    if (field == WHB_OUT) WHB_TRY(ensure_out(c, member));
    WHB_TRY(copy_field_d2h(c, field_ptr(c, field, member), host));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
}

namespace {
// One 3D copy between a strided host view of the owned planes (element strides sp between
// storage planes and sr between rows, last axis contiguous) and the pitched device field.
int copy_field_strided(whb_ctx *c, double *dev, double *host, int64_t sp, int64_t sr, bool h2d) {
    const int64_t n1 = c->gshape[1], n2 = c->gshape[2];
    if (sr < n2 || (n1 > 1 && sp % sr) || sp < n1 * sr)
        return fail(WHB_E_ARG, "strided host view: row / plane strides do not describe the field");
    cudaMemcpy3DParms q = {};
    const size_t hpitch = (size_t)(n1 > 1 ? sr : sp) * sizeof(double);
    const size_t hrows = (size_t)(n1 > 1 ? sp / sr : 1);
    cudaPitchedPtr hp = make_cudaPitchedPtr(host, hpitch, (size_t)n2, hrows);
    cudaPitchedPtr dp = make_cudaPitchedPtr(owned(dev, c), (size_t)c->P * sizeof(double), (size_t)n2, (size_t)n1);
    q.srcPtr = h2d ? hp : dp;
    q.dstPtr = h2d ? dp : hp;
    q.extent = make_cudaExtent((size_t)n2 * sizeof(double), (size_t)n1, (size_t)c->nloc);
    q.kind = h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    WHB_CUDA(cudaMemcpy3DAsync(&q, c->stream));
    return 0;
}
}  // namespace

int whb_upload_strided(whb_ctx *c, int field, int member, const double *host, int64_t plane_stride,
                       int64_t row_stride) {
    if (!c || !host) return fail(WHB_E_ARG, "NULL argument");
    if (member < 0 || member >= c->nbatch || field < 0 || field > WHB_WD) return fail(WHB_E_ARG, "bad field/member");
    WHB_TRY(set_dev(c));
    if (field == WHB_OUT) WHB_TRY(ensure_out(c, member));
    double *d = field_ptr(c, field, member);
    WHB_TRY(copy_field_strided(c, d, const_cast<double *>(host), plane_stride, row_stride, true));
    WHB_TRY(zero_bnd(c, d));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
}

int whb_download_strided(whb_ctx *c, int field, int member, double *host, int64_t plane_stride, int64_t row_stride) {
    if (!c || !host) return fail(WHB_E_ARG, "NULL argument");
    if (member < 0 || member >= c->nbatch || field < 0 || field > WHB_WD) return fail(WHB_E_ARG, "bad field/member");
    WHB_TRY(set_dev(c));
    if (field == WHB_OUT) WHB_TRY(ensure_out(c, member));
    WHB_TRY(copy_field_strided(c, field_ptr(c, field, member), host, plane_stride, row_stride, false));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
}

int whb_zero(whb_ctx *c, int field, int member) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (member < 0 || member >= c->nbatch || field < 0 || field > WHB_WD) return fail(WHB_E_ARG, "bad field/member");
    WHB_TRY(set_dev(c));
    if (field == WHB_OUT) WHB_TRY(ensure_out(c, member));
    WHB_CUDA(cudaMemsetAsync(field_ptr(c, field, member), 0, (size_t)c->field_elems * sizeof(double), c->stream));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
}

int whb_filtered_solve(whb_ctx *c, int out_mode, int zero_forcing, double *resid_sq) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (out_mode < 0 || out_mode > 2) return fail(WHB_E_ARG, "bad out_mode");
    WHB_TRY(set_dev(c));
    WHB_TRY(check_ready(c));
    const int zf = (zero_forcing || out_mode == WHB_OUT_AV) ? 1 : 0;
    WHB_TRY(upload_members(c, out_mode, zf));
    if (out_mode == WHB_OUT_FPI) WHB_CUDA(cudaMemsetAsync(c->d_counter, 0, sizeof(int), c->stream));
    if (c->timing) {
        WHB_TRY(ensure_events(c, 2));
        WHB_CUDA(cudaEventRecord(c->ev[0], c->stream));
    }
    WHB_TRY(run_solve(c, out_mode, zf));
    if (c->timing) WHB_CUDA(cudaEventRecord(c->ev[1], c->stream));
    if (out_mode == WHB_OUT_FPI && resid_sq)
        WHB_CUDA(cudaMemcpyAsync(resid_sq, c->d_hist, c->nbatch * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    if (c->timing) {
        float ms = 0.f;
        WHB_CUDA(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
        c->t_solve_ms = ms;
        c->t_step_ms = ms;
        c->t_step_launches = max_steps(c);
    }
    return 0;
}

int whb_fpi(whb_ctx *c, int iters, double tol_sq, double *resid_sq_out, int *iters_done) {
    if (!c || iters < 0) return fail(WHB_E_ARG, "bad argument");
    WHB_TRY(set_dev(c));
    if (iters == 0) {
        if (iters_done) *iters_done = 0;
        return 0;
    }
    return fpi_impl(c, iters, tol_sq, resid_sq_out, iters_done);
}

int whb_fpi_scaled(whb_ctx *c, int iters, double tol, double root_n, double *resid_sq_out, int *iters_done) {
    if (!c || iters < 0 || !(root_n > 0.0)) return fail(WHB_E_ARG, "bad argument");
    WHB_TRY(set_dev(c));
    if (iters == 0) {
        if (iters_done) *iters_done = 0;
        return 0;
    }
    return fpi_impl(c, iters, -1.0, resid_sq_out, iters_done, tol, root_n);
}

// whb_iterate_host on the three-step plan (whole-grid 3D, Dirichlet): the host transfers are hidden
// behind the passes.  The grid is cut into bands of rows (axis 1; a multiple of the 12-row tiles).
// Band b of v is uploaded on a copy-in stream (one strided copy + a re-pitch kernel that also
// zeroes the boundary); on the context stream the (pass p, band b) launches are enqueued by
// diagonals d = p + b, passes ascending inside a diagonal.  Pass p on band b reads what pass p-1
// wrote on bands b-1, b, b+1 (a k-step pass reaches k <= 3 rows past its band) -- diagonals
// d-2, d-1 and, earlier in the same diagonal, (p-1, b+1); a level-ring slot written by (q, b) was
// last read by (q-2, b+1) at most, an earlier diagonal.  Band b of the new v leaves on a copy-out
// stream as soon as the last pass has run on it.  Per launch: one wave of CTAs (17 x 1 x nch main
// tiles + the edge tiles <= 148 SMs), axis-0 chunks chosen for that.  The passes are the plan's
// (three-step passes, then one or two two-step passes for the remainder); every step is the same
// arithmetic as in the whole-grid launches, so the iterate is bitwise the same, and the residual
// sums the same squares in another order.  WHB_PIPE=0 keeps the serial path (upload, solve graph,
// download); WHB_PIPE_ROWS sets the band height in tiles.
struct HostView {  // a host field as (planes, rows, n2) with element strides (C-contiguous: n1 * n2, n2)
    double *p;
    int64_t plane_stride, row_stride;
};

int solve_host_banded(whb_ctx *c, HostView vin, HostView vout, int out_mode, int zf, double *resid_sq, bool *done) {
    *done = false;
    static const bool off = getenv("WHB_PIPE") && std::string(getenv("WHB_PIPE")) == "0";
    const int ns = max_steps(c);
    const int n0 = (int)c->gshape[0], n1 = (int)c->gshape[1], n2 = (int)c->gshape[2];
    if (off || !c->t3 || !c->tb2 || c->kern != 2 || c->nbatch != 1 || !c->act0 || !c->act1 || ns < 9 ||
        c->plane_begin != 0 || c->plane_end != c->gshape[0] || (int)c->nloc != n0 || cres_smem(c) || c->wfT)
        return 0;
    for (const HostView &h : {vin, vout})  // rows of n2 elements, planes of whole rows (cudaMemcpy3D pitched view)
        if (h.row_stride < n2 || h.plane_stride % h.row_stride || h.plane_stride < (int64_t)n1 * h.row_stride) return 0;
    // passes: three steps while the remainder stays 0, 2 or 4; then two-step passes
    struct Pass { int s, k; };
    std::vector<Pass> passes;
    int s = 0;
    while (ns - s >= 3 && (ns - s - 3) != 1) { passes.push_back({s, 3}); s += 3; }
    while (ns - s >= 2) { passes.push_back({s, 2}); s += 2; }
    if (s != ns) return 0;
    const int NP = (int)passes.size();
    // bands of tile rows: `bt` tiles high, ramping up from one tile at both ends (the pipeline fills
    // and drains in units of the band height: the first launches wait for the uploads, the last
    // downloads for the last launches); per band, axis-0 chunks so that a launch is one wave of CTAs
    int bt = 2;  // measured on config 4 (ms per call, 4 streams): 1 -> 495, 2 -> 436, 4 -> 511; serial path ~690
    if (const char *e = getenv("WHB_PIPE_ROWS")) bt = std::max(1, atoi(e));
    int ramp = 0;  // one-tile bands at each end, then doubling up to bt (measured: 0 -> 427 ms per call, 8 -> 443, 16 -> 468)
    if (const char *e = getenv("WHB_PIPE_RAMP")) ramp = std::max(0, atoi(e));
    const int rows_total = n1 - 1;  // rows 0 .. n1-2 carry tiles (row 0 and n1-1 are Dirichlet)
    const int tiles_total = (rows_total + t3::BY - 1) / t3::BY;
    struct Band { int t0, t1, cl3, cl2, lx, po; };
    std::vector<Band> bands;
    {
        std::vector<int> front;  // heights from one end: `ramp` bands of 1, then 2, 4, .. (`ramp` / 2 each) below bt
        for (int h = 1, n = ramp; h < bt && n > 0; h *= 2, n = std::max(1, n / 2))
            for (int q = 0; q < n; ++q) front.push_back(h);
        int fsum = 0;
        for (int h : front) fsum += h;
        if (2 * fsum > tiles_total) front.clear(), fsum = 0;
        std::vector<int> hs(front);
        int mid = tiles_total - 2 * fsum;
        while (mid > 0) { hs.push_back(std::min(bt, mid)); mid -= std::min(bt, mid); }
        hs.insert(hs.end(), front.rbegin(), front.rend());
        int t = 0;
        for (int h : hs) { bands.push_back({t, t + h, 0, 0, 0, 0}); t += h; }
    }
    const int NB = (int)bands.size();
    if (NB < 2) return 0;
    int sms = 0;
    WHB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    const int npl = c->upd_hi - c->upd_lo;
    const Pass &lastp = passes.back();
    int parts = 0;
    for (Band &B : bands) {
        const int h = B.t1 - B.t0;
        // edge tile shape of a band: a one-wave launch lasts as long as its slowest CTA, and the 124 x 4
        // shape stages 386 box rows per plane (the main shape 50): take the widest shape that still
        // covers the band's rows with one tile (28 x 28, 60 x 12, 124 x 4); WHB_PIPE_LXE forces one
        B.lx = c->lxe3;
        if (B.lx != 32) {
            const int rows = h * t3::BY;
            B.lx = rows <= t3::Shape<16>::BY ? 16 : rows <= t3::Shape<8>::BY ? 8 : 4;
            B.lx = std::max(B.lx, c->lxe3);  // not narrower than the remainder needs
            if (const char *e = getenv("WHB_PIPE_LXE")) {
                const int v = atoi(e);
                if ((v == 4 || v == 8 || v == 16) && v >= c->lxe3) B.lx = v;
            }
        }
        // (the edge column's h slots per chunk all run, as shorter chunks)
        const int nch3 = std::max(1, sms / std::max(1, c->gx3 * h));
        const int jt2 = (h * t3::BY + T3_BY - 1) / T3_BY;
        const int nch2 = std::max(1, sms / std::max(1, c->gx2 * jt2));
        B.cl3 = (npl + nch3 - 1) / nch3;
        B.cl2 = (npl + nch2 - 1) / nch2;
        B.po = parts;  // residual partial slots: the last pass writes one per CTA
        parts += lastp.k == 3 ? c->gx3 * h * ((npl + B.cl3 - 1) / B.cl3) : c->gx2 * jt2 * ((npl + B.cl2 - 1) / B.cl2);
    }
    if (parts > c->nparts) return 0;
    // small grids: a band's one-wave launch would cut the march into chunks too short to amortise a
    // CTA's start-up (~20 planes' worth); they keep the serial path unless WHB_PIPE=1 forces bands
    static const bool force = getenv("WHB_PIPE") && std::string(getenv("WHB_PIPE")) == "1";
    if (!force && bands[NB / 2].cl3 < 64) return 0;
    if (!c->s_in) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);  // the small copy kernels go first when an SM frees up
        WHB_CUDA(cudaStreamCreateWithPriority(&c->s_in, cudaStreamNonBlocking, hi));
        WHB_CUDA(cudaStreamCreateWithPriority(&c->s_out, cudaStreamNonBlocking, hi));
    }
    // pass launches run as a dataflow over NS streams, diagonal d on stream d % NS (a diagonal is a
    // chain: (p, b) needs (p-1, b+1), the launch before it): a launch also waits for the events of
    // (p-1, b) and (p-1, b-1) on the two previous diagonals, so neighbouring diagonals overlap and
    // the drain / fill gap between the dependent one-wave launches of one diagonal is covered by the
    // next diagonal's work.  WHB_PIPE_STREAMS=1: one stream.
    int NS = 2;  // measured on config 4 (ms per call): 1 -> 484, 2 -> 427, 4 -> 436
    if (const char *e = getenv("WHB_PIPE_STREAMS")) NS = std::max(1, std::min(16, atoi(e)));
    while ((int)c->s_band.size() < NS) {
        cudaStream_t st;
        WHB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        c->s_band.push_back(st);
    }
    // events: [0, NB) uploads, [NB, 3 NB) pass launches (p % 2, b), then one per stream, then the start
    const int EV_PASS = NB, EV_STREAM = 3 * NB, EV_START = 3 * NB + NS;
    while ((int)c->ev_band.size() < EV_START + 1) {
        cudaEvent_t e;
        WHB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_band.push_back(e);
    }
    const bool fpi = out_mode == WHB_OUT_FPI;
    WHB_TRY(ensure_hist(c, 1));
    WHB_TRY(upload_members(c, out_mode, zf));
    if (fpi) WHB_CUDA(cudaMemsetAsync(c->d_counter, 0, sizeof(int), c->stream));
    c->cur_zf = zf;
    double *v = c->mem[0].v;
    double *result = fpi ? v : c->mem[0].out;  // W(v, f) replaces v, or goes to the output field
    auto band = [&](int b, int &ja, int &jb) {
        ja = bands[b].t0 * t3::BY;
        jb = b == NB - 1 ? n1 : std::min(n1, bands[b].t1 * t3::BY);  // copies: the last band takes row n1-1 too
    };
    // host <-> pitched device rows: one 3D copy per band (copy engines only; measured equal to a
    // contiguous copy into a staging field + a re-pitch kernel, which needs SMs the passes occupy)
    static const bool nocopy = getenv("WHB_PIPE_NOCOPY") != nullptr;  // timing experiments: passes only
    auto copy_band = [&](const HostView &h, double *dev, int ja, int jb, bool h2d, cudaStream_t st) -> int {
        if (nocopy) return 0;
        cudaMemcpy3DParms q = {};
        cudaPitchedPtr hp = make_cudaPitchedPtr(h.p, (size_t)h.row_stride * sizeof(double), (size_t)n2,
                                                (size_t)(h.plane_stride / h.row_stride));
        cudaPitchedPtr dp = make_cudaPitchedPtr(owned(dev, c), (size_t)c->P * sizeof(double), (size_t)n2, (size_t)n1);
        q.srcPtr = h2d ? hp : dp;
        q.dstPtr = h2d ? dp : hp;
        q.srcPos = make_cudaPos(0, (size_t)ja, 0);
        q.dstPos = make_cudaPos(0, (size_t)ja, 0);
        q.extent = make_cudaExtent((size_t)n2 * sizeof(double), (size_t)(jb - ja), (size_t)n0);
        q.kind = h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
        WHB_CUDA(cudaMemcpy3DAsync(&q, st));
        return 0;
    };
    cudaEvent_t ev0 = c->ev_band[EV_START];
    static const bool trace = getenv("WHB_PIPE_TRACE") != nullptr;  // stderr: upload / compute / download end times
    cudaEvent_t tev[4] = {};
    if (trace) {
        for (auto &e : tev) WHB_CUDA(cudaEventCreate(&e));
        WHB_CUDA(cudaEventRecord(tev[0], c->stream));
    }
    WHB_CUDA(cudaEventRecord(ev0, c->stream));
    WHB_CUDA(cudaStreamWaitEvent(c->s_in, ev0, 0));
    WHB_CUDA(cudaStreamWaitEvent(c->s_out, ev0, 0));
    for (int q = 0; q < NS; ++q) WHB_CUDA(cudaStreamWaitEvent(c->s_band[q], ev0, 0));
    cudaStream_t main_stream = c->stream;
    for (int b = 0; b < NB; ++b) {
        int ja, jb;
        band(b, ja, jb);
        WHB_TRY(copy_band(vin, v, ja, jb, true, c->s_in));
        band_zero_kernel<<<74, 256, 0, c->s_in>>>(owned(v, c), n0, n1, n2, c->P, c->S0, ja, jb);
        c->launches++;
        WHB_CUDA(cudaGetLastError());
        WHB_CUDA(cudaEventRecord(c->ev_band[b], c->s_in));
    }
    if (trace) WHB_CUDA(cudaEventRecord(tev[1], c->s_in));
    const auto h0 = std::chrono::steady_clock::now();
    int rc = 0;
    static const bool trace2 = trace && std::string(getenv("WHB_PIPE_TRACE")) == "2";
    for (int d = 0; d < NB + NP - 1 && !rc; ++d) {
        if (trace2 && d % 8 == 0)
            fprintf(stderr, "[whb banded] diagonal %d enqueued at host %.2f ms (%lld launches)\n", d,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count(),
                    (long long)c->launches);
        for (int p = 0; p < NP && !rc; ++p) {
            const int b = d - p;
            if (b < 0 || b >= NB) continue;
            cudaStream_t st = c->s_band[d % NS];
            if (p == 0) {
                WHB_CUDA(cudaStreamWaitEvent(st, c->ev_band[std::min(b + 1, NB - 1)], 0));
            } else if (NS > 1) {  // (p-1, b+1) is the launch before this one on the diagonal's stream
                const int base = EV_PASS + ((p - 1) & 1) * NB;
                WHB_CUDA(cudaStreamWaitEvent(st, c->ev_band[base + b], 0));
                if (b > 0) WHB_CUDA(cudaStreamWaitEvent(st, c->ev_band[base + b - 1], 0));
            }
            c->stream = st;  // the launchers enqueue on the context stream
            const bool last = (p == NP - 1);
            const Band &B = bands[b];
            c->win_j0 = B.t0 * t3::BY;
            c->win_j1 = b == NB - 1 ? n1 : B.t1 * t3::BY;
            c->win_po = last ? B.po : 0;
            c->win_lxe = B.lx;
            if (passes[p].k == 3) rc = launch_t3(c, passes[p].s, last, c->upd_lo, c->upd_hi, B.cl3);
            else rc = launch_pair_range(c, passes[p].s, c->upd_lo, c->upd_hi, B.cl2, c->win_po);
            c->stream = main_stream;
            cudaEvent_t evp = c->ev_band[EV_PASS + (p & 1) * NB + b];
            if (!rc) WHB_CUDA(cudaEventRecord(evp, st));
            if (last && !rc) {
                int ja, jb;
                band(b, ja, jb);
                WHB_CUDA(cudaStreamWaitEvent(c->s_out, evp, 0));
                WHB_TRY(copy_band(vout, result, ja, jb, false, c->s_out));
            }
        }
    }
    c->win_j0 = 0;
    c->win_j1 = INT_MAX;
    c->win_po = 0;
    c->win_lxe = 0;
    for (int q = 0; q < NS; ++q) {  // the context stream continues after every band stream
        cudaEventRecord(c->ev_band[EV_STREAM + q], c->s_band[q]);
        cudaStreamWaitEvent(c->stream, c->ev_band[EV_STREAM + q], 0);
    }
    if (rc) {
        cudaStreamSynchronize(c->s_in);
        cudaStreamSynchronize(c->stream);
        cudaStreamSynchronize(c->s_out);
        return rc;
    }
    if (fpi) {
        reduce_partials_kernel<<<1, 1024, 0, c->stream>>>(c->d_members, 1, parts, c->d_hist, c->d_counter);
        c->launches++;
        WHB_CUDA(cudaGetLastError());
        if (resid_sq) WHB_CUDA(cudaMemcpyAsync(resid_sq, c->d_hist, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    }
    const double host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
    if (trace) {
        WHB_CUDA(cudaEventRecord(tev[2], c->stream));
        WHB_CUDA(cudaEventRecord(tev[3], c->s_out));
    }
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    WHB_CUDA(cudaStreamSynchronize(c->s_out));
    if (trace) {
        float up = 0.f, comp = 0.f, down = 0.f;
        cudaEventElapsedTime(&up, tev[0], tev[1]);
        cudaEventElapsedTime(&comp, tev[0], tev[2]);
        cudaEventElapsedTime(&down, tev[0], tev[3]);
        fprintf(stderr, "[whb banded] bands %d x passes %d: upload done %.1f ms, passes done %.1f ms, download done %.1f ms; "
                "host enqueue of the passes %.1f ms (chunks of %d planes)\n", NB, NP, up, comp, down, host_ms,
                bands[NB / 2].cl3);
        for (auto &e : tev) cudaEventDestroy(e);
    }
    *done = true;
    return 0;
}

int whb_iterate_host(whb_ctx *c, const double *v_host, double *v_out_host, double *resid_sq) {
    if (!c || !v_host || !v_out_host) return fail(WHB_E_ARG, "NULL argument");
    if (c->nbatch != 1) return fail(WHB_E_ARG, "whb_iterate_host needs nbatch == 1");
    WHB_TRY(set_dev(c));
    WHB_TRY(check_ready(c));
    bool banded = false;
    const int64_t hp = c->gshape[1] * c->gshape[2], hr = c->gshape[2];
    WHB_TRY(solve_host_banded(c, HostView{const_cast<double *>(v_host), hp, hr}, HostView{v_out_host, hp, hr},
                              WHB_OUT_FPI, 0, resid_sq, &banded));
    if (banded) return 0;
    WHB_TRY(ensure_hist(c, 1));
    WHB_TRY(upload_members(c, WHB_OUT_FPI, 0));
    WHB_TRY(copy_field_h2d(c, c->mem[0].v, v_host));
    WHB_TRY(zero_bnd(c, c->mem[0].v));
    WHB_CUDA(cudaMemsetAsync(c->d_counter, 0, sizeof(int), c->stream));
    WHB_TRY(run_solve(c, WHB_OUT_FPI, 0));
    WHB_TRY(copy_field_d2h(c, c->mem[0].v, v_out_host));
    if (resid_sq) WHB_CUDA(cudaMemcpyAsync(resid_sq, c->d_hist, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
}

int whb_solve_host(whb_ctx *c, const double *v_host, int64_t v_plane_stride, int64_t v_row_stride, double *out_host,
                   int64_t out_plane_stride, int64_t out_row_stride, int out_mode, int zero_forcing, double *resid_sq) {
    if (!c || !v_host || !out_host) return fail(WHB_E_ARG, "NULL argument");
    if (out_mode < 0 || out_mode > 2) return fail(WHB_E_ARG, "bad out_mode");
    if (c->nbatch != 1) return fail(WHB_E_ARG, "whb_solve_host needs nbatch == 1");
    WHB_TRY(set_dev(c));
    WHB_TRY(check_ready(c));
    const int zf = (zero_forcing || out_mode == WHB_OUT_AV) ? 1 : 0;
    bool banded = false;
    WHB_TRY(solve_host_banded(c, HostView{const_cast<double *>(v_host), v_plane_stride, v_row_stride},
                              HostView{out_host, out_plane_stride, out_row_stride}, out_mode, zf, resid_sq, &banded));
    if (banded) return 0;
    // serial path: upload, the solve graph, download
    double *v = c->mem[0].v;
    WHB_TRY(copy_field_strided(c, v, const_cast<double *>(v_host), v_plane_stride, v_row_stride, true));
    WHB_TRY(zero_bnd(c, v));
    WHB_TRY(ensure_hist(c, 1));
    WHB_TRY(upload_members(c, out_mode, zf));
    if (out_mode == WHB_OUT_FPI) WHB_CUDA(cudaMemsetAsync(c->d_counter, 0, sizeof(int), c->stream));
    WHB_TRY(run_solve(c, out_mode, zf));
    WHB_TRY(copy_field_strided(c, out_mode == WHB_OUT_FPI ? v : c->mem[0].out, out_host, out_plane_stride,
                               out_row_stride, false));
    if (out_mode == WHB_OUT_FPI && resid_sq)
        WHB_CUDA(cudaMemcpyAsync(resid_sq, c->d_hist, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
}

// ---- vectors -------------------------------------------------------------------------------

int whb_vec_reserve(whb_ctx *c, int count, int *first_id) {
    if (!c || count < 0) return fail(WHB_E_ARG, "bad argument");
    WHB_TRY(set_dev(c));
    const int first = 8 + (int)c->vecs.size();
    for (int i = 0; i < count; ++i) {
        double *p = nullptr;
        WHB_TRY(alloc_field(c, &p));
        c->vecs.push_back(p);
    }
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    if (first_id) *first_id = first;
    return 0;
}

#define VEC_OR_FAIL(name, id)                                             \
    double *name = vec_ptr(c, id);                                        \
    if (!name) {                                                          \
        if ((id) == WHB_OUT) {                                            \
            WHB_TRY(ensure_out(c, 0));                                    \
            name = vec_ptr(c, id);                                        \
        } else                                                            \
            return fail(WHB_E_ARG, "unknown vector id " + std::to_string(id)); \
    }

int whb_vec_upload(whb_ctx *c, int id, const double *host) {
    if (!c || !host) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(x, id);
    WHB_TRY(copy_field_h2d(c, x, host));
    WHB_TRY(zero_bnd(c, x));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
}

int whb_vec_download(whb_ctx *c, int id, double *host) {
    if (!c || !host) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(x, id);
    WHB_TRY(copy_field_d2h(c, x, host));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
}

int whb_vec_dot(whb_ctx *c, int xi, int yi, double *out) {
    if (!c || !out) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(x, xi);
    VEC_OR_FAIL(y, yi);
    return vec_reduce_dot(c, x, y, out);
}

#define ELEMWISE_LAUNCH(kernel, ...)                                                 \
    do {                                                                            \
        kernel<<<kRedBlocks, kRedThreads, 0, c->stream>>>(__VA_ARGS__);             \
        c->launches++;                                                              \
        WHB_CUDA(cudaGetLastError());                                               \
    } while (0)

int whb_vec_axpy(whb_ctx *c, double a, int xi, int yi) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(x, xi);
    VEC_OR_FAIL(y, yi);
    // y - ((-a)*x) == y + a*x bitwise; with a = -h this is numpy's `w -= h*q` (linalg.py:146)
    ELEMWISE_LAUNCH(axmy_kernel, -a, owned(x, c), owned(y, c), owned_elems(c));
    return 0;
}

int whb_vec_scale_into(whb_ctx *c, double a, int xi, int yi) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(x, xi);
    VEC_OR_FAIL(y, yi);
    ELEMWISE_LAUNCH(scale_kernel, a, owned(x, c), owned(y, c), owned_elems(c));
    return 0;
}

int whb_vec_div_into(whb_ctx *c, int xi, double d, int yi) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(x, xi);
    VEC_OR_FAIL(y, yi);
    ELEMWISE_LAUNCH(div_kernel, owned(x, c), d, owned(y, c), owned_elems(c));
    return 0;
}

int whb_vec_sub_into(whb_ctx *c, int xi, int yi, int zi) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(x, xi);
    VEC_OR_FAIL(y, yi);
    VEC_OR_FAIL(z, zi);
    ELEMWISE_LAUNCH(sub_kernel, owned(x, c), owned(y, c), owned(z, c), owned_elems(c));
    return 0;
}

int whb_vec_copy(whb_ctx *c, int xi, int yi) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(x, xi);
    VEC_OR_FAIL(y, yi);
    WHB_CUDA(cudaMemcpyAsync(y, x, (size_t)c->field_elems * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    return 0;
}

int whb_vec_lincomb(whb_ctx *c, int yi, int first, int count, const double *coef) {
    if (!c || (!coef && count > 0)) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(y, yi);
    for (int base = 0; base < count; base += kMaxComb) {
        // NB: chunks of 64 add their partial sums to y separately; GMRES restarts are <= 64 in practice
        CombArgs a{};
        const int cnt = std::min(kMaxComb, count - base);
        for (int j = 0; j < cnt; ++j) {
            double *q = vec_ptr(c, first + base + j);
            if (!q) return fail(WHB_E_ARG, "unknown vector id in lincomb");
            a.q[j] = owned(q, c);
            a.c[j] = coef[base + j];
        }
        ELEMWISE_LAUNCH(lincomb_kernel, a, cnt, owned(y, c), owned_elems(c));
    }
    return 0;
}

int whb_matvec(whb_ctx *c, int xi, int yi) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (c->nbatch != 1) return fail(WHB_E_ARG, "whb_matvec needs nbatch == 1");
    if (xi == yi) return fail(WHB_E_ARG, "whb_matvec needs distinct x and y");
    WHB_TRY(set_dev(c));
    WHB_TRY(check_ready(c));
    VEC_OR_FAIL(x, xi);
    VEC_OR_FAIL(y, yi);
    const MemberHost &h0 = c->mem[0];
    bool alias = (x == h0.acc || y == h0.acc);
    for (int q = 0; q < 6; ++q) alias = alias || x == h0.ring[q] || y == h0.ring[q];
    if (alias)
        return fail(WHB_E_ARG, "whb_matvec operands may not alias the leapfrog workspace");
    WHB_TRY(upload_members(c, WHB_OUT_AV, 1, x, y));
    WHB_TRY(run_solve(c, WHB_OUT_AV, 1));
    return 0;
}

int whb_apply_operator(whb_ctx *c, int xi, int yi) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (xi == yi) return fail(WHB_E_ARG, "whb_apply_operator needs distinct x and y");
    WHB_TRY(set_dev(c));
    if (!c->op_set) return fail(WHB_E_STATE, "operator not set (whb_set_operator)");
    VEC_OR_FAIL(x, xi);
    VEC_OR_FAIL(y, yi);
    if (c->kern == 3) {
        apply_general_kernel<<<kGenBlocks, 256, 0, c->stream>>>(c->geomg, x, y, (int)c->nloc);
        c->launches++;
        WHB_CUDA(cudaGetLastError());
        return 0;
    }
    // update planes exclude global Dirichlet planes; ghost planes of x must hold neighbour data
    apply_operator_kernel<<<kRedBlocks, kRedThreads, 0, c->stream>>>(c->geom, x, y, c->act0, c->act1, c->upd_lo,
                                                                     c->upd_hi);
    c->launches++;
    WHB_CUDA(cudaGetLastError());
    return 0;
}

// ---- slab step-level control ----------------------------------------------------------------

int whb_solve_begin(whb_ctx *c, int out_mode, int zero_forcing) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (c->nbatch != 1) return fail(WHB_E_ARG, "step-level control needs nbatch == 1");
    WHB_TRY(set_dev(c));
    WHB_TRY(check_ready(c));
    WHB_TRY(ensure_hist(c, 1));
    const int zf = (zero_forcing || out_mode == WHB_OUT_AV) ? 1 : 0;
    WHB_TRY(upload_members(c, out_mode, zf));
    if (out_mode == WHB_OUT_FPI) {
        WHB_CUDA(cudaMemsetAsync(c->d_counter, 0, sizeof(int), c->stream));
        // region-split launches leave some partial slots unwritten: start from zero
        WHB_CUDA(cudaMemsetAsync(c->mem[0].partials, 0, (size_t)c->nparts * sizeof(double), c->stream));
    }
    c->cur_mode = out_mode;
    c->cur_zf = zf;
    c->cur_parts = 0;
    return 0;
}

int whb_step(whb_ctx *c, int s, int region) {
    if (!c || c->cur_mode < 0) return fail(WHB_E_STATE, "whb_step outside whb_solve_begin/end");
    if (s < 0 || s >= c->mem[0].n_total) return fail(WHB_E_ARG, "step out of range");
    WHB_TRY(set_dev(c));
    const int lo = c->upd_lo, hi = c->upd_hi;
    const int tiles = c->gx * c->JT;
    if (region == 0) {
        WHB_TRY(launch_step(c, s, 1, lo, hi, c->chunk_len, 0));
        if (s == c->mem[0].n_total - 1) c->cur_parts = tiles * c->nchunks;
    } else if (region == 1) {
        // the first and last owned update planes (what neighbours need), one plane per launch
        WHB_TRY(launch_step(c, s, 1, lo, std::min(lo + 1, hi), 1, 0));
        if (hi - 1 > lo) WHB_TRY(launch_step(c, s, 1, hi - 1, hi, 1, tiles));
    } else if (region == 2) {
        if (hi - 1 > lo + 1) WHB_TRY(launch_step(c, s, 1, lo + 1, hi - 1, c->chunk_len, 2 * tiles));
        if (s == c->mem[0].n_total - 1) c->cur_parts = c->nparts;
    } else
        return fail(WHB_E_ARG, "region must be 0, 1 or 2");
    return 0;
}

int whb_pair(whb_ctx *c, int s, int region) {
    if (!c || c->cur_mode < 0) return fail(WHB_E_STATE, "whb_pair outside whb_solve_begin/end");
    if (!c->tb2 || c->wfT) return fail(WHB_E_STATE, "context has no two-step plan (whb_plan)");
    if (s < 0 || s + 1 >= c->mem[0].n_total) return fail(WHB_E_ARG, "steps (s, s+1) out of range");
    WHB_TRY(set_dev(c));
    const int lo = c->upd_lo, hi = c->upd_hi;
    const bool last = s + 2 == c->mem[0].n_total;
    if (region == 0) {
        WHB_TRY(launch_pair_range(c, s, lo, hi, c->chunk2, 0));
        if (last) c->cur_parts = c->gx2 * c->JT2 * c->nch2;
    } else if (region == 1) {
        if (last) return fail(WHB_E_ARG, "the last pass runs as region 0 (nothing needs its halo)");
        // the two first and two last update planes: W^{s+2} there feeds the neighbours' 2 ghost planes
        if (hi - lo <= 4) {
            WHB_TRY(launch_pair_range(c, s, lo, hi, hi - lo, 0));
        } else {
            WHB_TRY(launch_pair_range(c, s, lo, lo + 2, 2, 0));
            WHB_TRY(launch_pair_range(c, s, hi - 2, hi, 2, 0));
        }
    } else if (region == 2) {
        if (last) return fail(WHB_E_ARG, "the last pass runs as region 0 (nothing needs its halo)");
        if (hi - lo > 4) {
            const int n = hi - lo - 4;
            const int cl = std::min(n, c->chunk2);
            WHB_TRY(launch_pair_range(c, s, lo + 2, hi - 2, cl, 0));
        }
    } else
        return fail(WHB_E_ARG, "region must be 0, 1 or 2");
    return 0;
}

int whb_triple(whb_ctx *c, int s, int region) {
    if (!c || c->cur_mode < 0) return fail(WHB_E_STATE, "whb_triple outside whb_solve_begin/end");
    if (!c->t3) return fail(WHB_E_STATE, "context has no three-step plan (whb_plan)");
    const int N = c->mem[0].n_total;
    if (s < 0 || s + 2 >= N) return fail(WHB_E_ARG, "steps (s, s+1, s+2) out of range");
    if (s == 0 && N == 3) return fail(WHB_E_ARG, "a three-step pass may not be both the first and the last");
    WHB_TRY(set_dev(c));
    const int lo = c->upd_lo, hi = c->upd_hi;
    const bool last = s + 3 == N;
    if (region == 0) {
        WHB_TRY(launch_t3(c, s, last, lo, hi, c->chunk3));
        if (last) c->cur_parts = c->gx3 * c->JT3 * ((hi - lo + c->chunk3 - 1) / c->chunk3);
    } else if (region == 1) {
        if (last) return fail(WHB_E_ARG, "the last pass runs as region 0 (nothing needs its halo)");
        // the three first and three last update planes: W^{s+3} there feeds the neighbours' 3 ghost planes
        if (hi - lo <= 6) {
            WHB_TRY(launch_t3(c, s, false, lo, hi, hi - lo));
        } else {
            WHB_TRY(launch_t3(c, s, false, lo, lo + 3, 3));
            WHB_TRY(launch_t3(c, s, false, hi - 3, hi, 3));
        }
    } else if (region == 2) {
        if (last) return fail(WHB_E_ARG, "the last pass runs as region 0 (nothing needs its halo)");
        if (hi - lo > 6) WHB_TRY(launch_t3(c, s, false, lo + 3, hi - 3, std::min(hi - lo - 6, c->chunk3)));
    } else
        return fail(WHB_E_ARG, "region must be 0, 1 or 2");
    return 0;
}

int whb_ghost_planes(whb_ctx *c, int *ghost) {
    if (!c || !ghost) return fail(WHB_E_ARG, "NULL argument");
    *ghost = GH;
    return 0;
}

int whb_field_plane_ptr(whb_ctx *c, int field, int member, int64_t plane, uint64_t *dev_ptr, int64_t *plane_elems) {
    if (!c || !dev_ptr) return fail(WHB_E_ARG, "NULL argument");
    if (member < 0 || member >= c->nbatch) return fail(WHB_E_ARG, "member out of range");
    if (plane < 0 || plane >= c->nplanes) return fail(WHB_E_ARG, "plane out of range");
    double *base = field_ptr(c, field, member);
    if (field == WHB_OUT) {
        WHB_TRY(set_dev(c));
        WHB_TRY(ensure_out(c, member));
        base = c->mem[member].out;
    }
    if (!base) return fail(WHB_E_ARG, "unknown field");
    *dev_ptr = (uint64_t)(uintptr_t)(base + plane * c->S0);
    if (plane_elems) *plane_elems = c->S0;
    return 0;
}

int whb_solve_end(whb_ctx *c, double *resid_sq) {
    if (!c || c->cur_mode < 0) return fail(WHB_E_STATE, "whb_solve_end without whb_solve_begin");
    WHB_TRY(set_dev(c));
    if (c->cur_mode == WHB_OUT_FPI) {
        // unused partial slots of region launches stay 0 from the previous zeroing
        reduce_partials_kernel<<<1, 1024, 0, c->stream>>>(c->d_members, 1, c->cur_parts, c->d_hist, c->d_counter);
        c->launches++;
        WHB_CUDA(cudaGetLastError());
        if (c->capturing) {  // the residual stays on the device (whb_resid_read after the replay)
            c->cur_mode = -1;
            if (resid_sq) *resid_sq = 0.0;
            return 0;
        }
        if (resid_sq) WHB_CUDA(cudaMemcpyAsync(resid_sq, c->d_hist, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    }
    if (c->capturing) {
        c->cur_mode = -1;
        return 0;
    }
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    c->cur_mode = -1;
    return 0;
}

int whb_capture_begin(whb_ctx *c) {
    if (!c || c->capturing) return fail(WHB_E_STATE, "capture already active");
    WHB_TRY(set_dev(c));
    WHB_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
    c->capturing = true;
    return 0;
}

int whb_capture_end(whb_ctx *c, int *graph_id) {
    if (!c || !c->capturing || !graph_id) return fail(WHB_E_STATE, "no capture active");
    WHB_TRY(set_dev(c));
    c->capturing = false;
    cudaGraph_t g;
    WHB_CUDA(cudaStreamEndCapture(c->stream, &g));
    cudaGraphExec_t ge;
    cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(WHB_E_CUDA, std::string("instantiate: ") + cudaGetErrorString(e));
    c->user_graphs.push_back(ge);
    *graph_id = (int)c->user_graphs.size() - 1;
    return 0;
}

int whb_graph_launch(whb_ctx *c, int graph_id) {
    if (!c || graph_id < 0 || graph_id >= (int)c->user_graphs.size()) return fail(WHB_E_ARG, "bad graph id");
    if (!c->user_graphs[graph_id])
        return fail(WHB_E_STATE, "graph invalidated (a buffer it baked was reallocated); capture it again");
    WHB_TRY(set_dev(c));
    WHB_CUDA(cudaGraphLaunch(c->user_graphs[graph_id], c->stream));
    return 0;
}

int whb_resid_read(whb_ctx *c, double *resid_sq) {
    if (!c || !resid_sq) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    WHB_CUDA(cudaMemcpyAsync(resid_sq, c->d_hist, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
}

int whb_level_plane_ptr(whb_ctx *c, int level, int64_t plane, uint64_t *dev_ptr, int64_t *plane_elems) {
    if (!c || !dev_ptr) return fail(WHB_E_ARG, "NULL argument");
    if (plane < 0 || plane >= c->nplanes) return fail(WHB_E_ARG, "plane out of range");
    if (level < 0) return fail(WHB_E_ARG, "level must be >= 0");
    const MemberHost &m = c->mem[0];
    const double *base = (level == 0) ? (c->cur_mode >= 0 && !c->h_members.empty() ? c->h_members[0].v : m.v)
                                      : m.ring[level % c->nring];
    *dev_ptr = (uint64_t)(uintptr_t)(base + plane * c->S0);
    if (plane_elems) *plane_elems = c->S0;
    return 0;
}

int whb_stream_ptr(whb_ctx *c, uint64_t *stream) {
    if (!c || !stream) return fail(WHB_E_ARG, "NULL argument");
    *stream = (uint64_t)(uintptr_t)c->stream;
    return 0;
}

int whb_synchronize(whb_ctx *c) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
}

int whb_copy_device(whb_ctx *src, uint64_t src_ptr, whb_ctx *dst, uint64_t dst_ptr, int64_t bytes) {
    if (!src || !dst || !src_ptr || !dst_ptr) return fail(WHB_E_ARG, "NULL argument");
    if (bytes <= 0) return 0;
    cudaEvent_t e1, e2;
    WHB_TRY(set_dev(src));
    WHB_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
    WHB_CUDA(cudaEventRecord(e1, src->stream));
    WHB_TRY(set_dev(dst));
    WHB_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
    WHB_CUDA(cudaStreamWaitEvent(dst->stream, e1, 0));
    WHB_CUDA(cudaMemcpyPeerAsync((void *)(uintptr_t)dst_ptr, dst->device, (const void *)(uintptr_t)src_ptr,
                                 src->device, (size_t)bytes, dst->stream));
    WHB_CUDA(cudaEventRecord(e2, dst->stream));
    WHB_TRY(set_dev(src));
    WHB_CUDA(cudaStreamWaitEvent(src->stream, e2, 0));
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    return 0;
}

// ---- peer-memory halo exchange (slab.PeerHalo): CUDA IPC mappings, copies and stream flags ----

namespace {
PFN_cuStreamWriteValue32_v11070 g_write32 = nullptr;
PFN_cuStreamWaitValue32_v11070 g_wait32 = nullptr;
PFN_cuMemGetAddressRange_v3020 g_addr_range = nullptr;

int get_memops() {
    if (g_write32 && g_wait32 && g_addr_range) return 0;
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
        return fail(WHB_E_CUDA, "cuStreamWriteValue32 entry point unavailable");
    g_write32 = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
        return fail(WHB_E_CUDA, "cuStreamWaitValue32 entry point unavailable");
    g_wait32 = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
        return fail(WHB_E_CUDA, "cuMemGetAddressRange entry point unavailable");
    g_addr_range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
    return 0;
}
}  // namespace

int whb_ipc_handle(whb_ctx *c, uint64_t dev_ptr, void *handle_out, int64_t *offset_out) {
    if (!c || !dev_ptr || !handle_out || !offset_out) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    WHB_TRY(get_memops());
    CUdeviceptr base = 0;
    size_t size = 0;
    if (g_addr_range(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS)
        return fail(WHB_E_ARG, "pointer is not inside a device allocation");
    cudaIpcMemHandle_t h;
    WHB_CUDA(cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base));
    memcpy(handle_out, &h, sizeof(h));
    *offset_out = (int64_t)(dev_ptr - (uint64_t)base);
    return 0;
}

int whb_ipc_open(whb_ctx *c, const void *handle, uint64_t *base_out) {
    if (!c || !handle || !base_out) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void *p = nullptr;
    WHB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    *base_out = (uint64_t)(uintptr_t)p;
    return 0;
}

int whb_ipc_close(whb_ctx *c, uint64_t base) {
    if (!c || !base) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    WHB_CUDA(cudaIpcCloseMemHandle((void *)(uintptr_t)base));
    return 0;
}

int whb_flags_alloc(whb_ctx *c, int count, uint64_t *dev_ptr) {
    if (!c || count <= 0 || !dev_ptr) return fail(WHB_E_ARG, "bad argument");
    WHB_TRY(set_dev(c));
    void *p = nullptr;
    WHB_CUDA(cudaMalloc(&p, (size_t)count * sizeof(uint32_t)));
    WHB_CUDA(cudaMemset(p, 0, (size_t)count * sizeof(uint32_t)));
    *dev_ptr = (uint64_t)(uintptr_t)p;
    return 0;
}

int whb_flags_free(whb_ctx *c, uint64_t dev_ptr) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    if (dev_ptr) WHB_CUDA(cudaFree((void *)(uintptr_t)dev_ptr));
    return 0;
}

int whb_copy_async(whb_ctx *c, uint64_t src_ptr, uint64_t dst_ptr, int64_t bytes) {
    if (!c || !src_ptr || !dst_ptr) return fail(WHB_E_ARG, "NULL argument");
    if (bytes <= 0) return 0;
    WHB_TRY(set_dev(c));
    WHB_CUDA(cudaMemcpyAsync((void *)(uintptr_t)dst_ptr, (const void *)(uintptr_t)src_ptr, (size_t)bytes,
                             cudaMemcpyDefault, c->on_comm ? c->comm : c->stream));
    return 0;
}

int whb_stream_write_u32(whb_ctx *c, uint64_t dev_ptr, uint32_t value) {
    if (!c || !dev_ptr) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    WHB_TRY(get_memops());
    // default flags: the write is preceded by a memory fence (earlier copies on the stream are visible first)
    if (g_write32((CUstream)(c->on_comm ? c->comm : c->stream), (CUdeviceptr)dev_ptr, value,
                  CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
        return fail(WHB_E_CUDA, "cuStreamWriteValue32 failed");
    return 0;
}

int whb_stream_wait_u32(whb_ctx *c, uint64_t dev_ptr, uint32_t value) {
    if (!c || !dev_ptr) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    WHB_TRY(get_memops());
    // (int32_t)(*addr - value) >= 0: wrap-safe monotone counters
    if (g_wait32((CUstream)c->stream, (CUdeviceptr)dev_ptr, value, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        return fail(WHB_E_CUDA, "cuStreamWaitValue32 failed");
    return 0;
}

int whb_comm_begin(whb_ctx *c) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (c->on_comm) return fail(WHB_E_STATE, "whb_comm_begin: exchange already open");
    static const bool off = getenv("WHB_COMM") && std::string(getenv("WHB_COMM")) == "0";
    if (off && !c->nccl) return 0;  // A/B switch: peer exchange on the context stream
    WHB_TRY(set_dev(c));
    if (!c->comm) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);  // the exchange gets the higher priority
        WHB_CUDA(cudaStreamCreateWithPriority(&c->comm, cudaStreamNonBlocking, hi));
        WHB_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        WHB_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
    WHB_CUDA(cudaEventRecord(c->ev_fork, c->stream));
    WHB_CUDA(cudaStreamWaitEvent(c->comm, c->ev_fork, 0));
    c->on_comm = true;
    return 0;
}

int whb_comm_end(whb_ctx *c) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (!c->on_comm) {
        static const bool off = getenv("WHB_COMM") && std::string(getenv("WHB_COMM")) == "0";
        if (off && !c->nccl) return 0;
        return fail(WHB_E_STATE, "whb_comm_end: no exchange open");
    }
    WHB_TRY(set_dev(c));
    c->on_comm = false;
    WHB_CUDA(cudaEventRecord(c->ev_join, c->comm));
    return 0;
}

int whb_comm_join(whb_ctx *c) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (!c->comm) return 0;
    WHB_TRY(set_dev(c));
    WHB_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    return 0;
}


int whb_nccl_unique_id(void *id_out) {
    if (!id_out) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(nccl_load());
    ncclUniqueId id;
    WHB_NCCL(g_nccl.get_unique_id(&id));
    std::memcpy(id_out, &id, sizeof(id));
    return 0;
}

int whb_nccl_init(whb_ctx *c, int nranks, int rank, const void *id) {
    if (!c || !id) return fail(WHB_E_ARG, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(WHB_E_ARG, "bad rank / nranks");
    if (c->nccl) return fail(WHB_E_STATE, "NCCL communicator already initialised");
    WHB_TRY(nccl_load());
    WHB_TRY(set_dev(c));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    WHB_NCCL(g_nccl.init_rank(&c->nccl, nranks, uid, rank));
    WHB_CUDA(cudaMalloc(&c->d_nccl, sizeof(double)));
    return 0;
}

int whb_nccl_exchange(whb_ctx *c, int n, const uint64_t *send_ptrs, const uint64_t *recv_ptrs, const int64_t *counts,
                      const int *peers) {
    if (!c || (n > 0 && (!send_ptrs || !recv_ptrs || !counts || !peers))) return fail(WHB_E_ARG, "NULL argument");
    if (!c->nccl) return fail(WHB_E_STATE, "whb_nccl_init first");
    if (!c->on_comm) return fail(WHB_E_STATE, "NCCL transfers go between whb_comm_begin and whb_comm_end");
    WHB_TRY(set_dev(c));
    WHB_NCCL(g_nccl.group_start());
    for (int i = 0; i < n; ++i) {
        if (counts[i] <= 0) continue;
        ncclResult_t r = g_nccl.send((const void *)(uintptr_t)send_ptrs[i], (size_t)counts[i], ncclDouble, peers[i],
                                     c->nccl, c->comm);
        if (r == ncclSuccess)
            r = g_nccl.recv((void *)(uintptr_t)recv_ptrs[i], (size_t)counts[i], ncclDouble, peers[i], c->nccl, c->comm);
        if (r != ncclSuccess) {
            g_nccl.group_end();
            return fail(WHB_E_CUDA, std::string("ncclSend/Recv: ") + g_nccl.err(r));
        }
    }
    WHB_NCCL(g_nccl.group_end());
    return 0;
}

int whb_nccl_allreduce_sum(whb_ctx *c, double *value) {
    if (!c || !value) return fail(WHB_E_ARG, "NULL argument");
    if (!c->nccl) return fail(WHB_E_STATE, "whb_nccl_init first");
    WHB_TRY(set_dev(c));
    WHB_CUDA(cudaMemcpyAsync(c->d_nccl, value, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    WHB_NCCL(g_nccl.all_reduce(c->d_nccl, c->d_nccl, 1, ncclDouble, ncclSum, c->nccl, c->stream));
    WHB_CUDA(cudaMemcpyAsync(value, c->d_nccl, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
}

int whb_copy_plane(whb_ctx *src, int src_level, int64_t src_plane, whb_ctx *dst, int dst_level, int64_t dst_plane) {
    if (!src || !dst) return fail(WHB_E_ARG, "NULL argument");
    if (src->S0 != dst->S0) return fail(WHB_E_ARG, "plane geometry mismatch");
    uint64_t sp = 0, dp = 0;
    WHB_TRY(whb_level_plane_ptr(src, src_level, src_plane, &sp, nullptr));
    WHB_TRY(whb_level_plane_ptr(dst, dst_level, dst_plane, &dp, nullptr));
    return whb_copy_device(src, sp, dst, dp, src->S0 * (int64_t)sizeof(double));
}

int whb_launch_count(whb_ctx *c, int64_t *count) {
    if (!c || !count) return fail(WHB_E_ARG, "NULL argument");
    *count = c->launches;
    return 0;
}

int whb_set_timing(whb_ctx *c, int enable) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    c->timing = enable != 0;
    return 0;
}

int whb_last_timing(whb_ctx *c, double *step_ms, int64_t *step_launches, double *solve_ms) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (step_ms) *step_ms = c->t_step_ms;
    if (step_launches) *step_launches = c->t_step_launches;
    if (solve_ms) *solve_ms = c->t_solve_ms;
    return 0;
}

int whb_set_l2_flush(whb_ctx *c, int64_t bytes) {
    if (!c || bytes < 0) return fail(WHB_E_ARG, "bad argument");
    WHB_TRY(set_dev(c));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(c->flush_buf);
    c->flush_buf = nullptr;
    c->flush_elems = 0;
    if (bytes > 0) {
        WHB_CUDA(cudaMalloc(&c->flush_buf, (size_t)bytes));
        c->flush_elems = bytes / (long long)sizeof(double);
    }
    return 0;
}

int whb_host_alloc(void **ptr, int64_t bytes) {
    if (!ptr || bytes < 0) return fail(WHB_E_ARG, "bad argument");
    WHB_CUDA(cudaMallocHost(ptr, (size_t)std::max<int64_t>(bytes, 8)));
    return 0;
}

int whb_host_free(void *ptr) {
    if (ptr) WHB_CUDA(cudaFreeHost(ptr));
    return 0;
}

int whb_plan(whb_ctx *c, int *kernel, int *steps_per_pass) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (kernel) *kernel = c->cres ? 4 : c->kern;
    if (steps_per_pass) *steps_per_pass = c->cres ? 0 : (c->wfT ? c->wfT : (c->t3 ? 3 : (c->tb2 ? 2 : 1)));
    return 0;
}

int whb_geometry(whb_ctx *c, int64_t *shape3, int64_t *pitch, int64_t *nloc) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (shape3)
        for (int a = 0; a < 3; ++a) shape3[a] = c->gshape[a];
    if (pitch) *pitch = c->P;
    if (nloc) *nloc = c->nloc;
    return 0;
}

// ---- implicit trapezoidal stepping ----------------------------------

int whb_imp_apply(whb_ctx *c, int xi, int yi, double s, int tmpi) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (xi == yi) return fail(WHB_E_ARG, "whb_imp_apply needs distinct x and y");
    WHB_TRY(set_dev(c));
    if (!c->op_set) return fail(WHB_E_STATE, "operator not set");
    VEC_OR_FAIL(x, xi);
    VEC_OR_FAIL(y, yi);
    double *t = nullptr;
    if (c->kern == 3) {  // general operator: t = c^2 L x (0 at boundaries), then y = x - s*t
        VEC_OR_FAIL(tv, tmpi);
        if (tv == x || tv == y) return fail(WHB_E_ARG, "whb_imp_apply scratch must differ from x and y");
        t = tv;
    }
    return imp_apply_enqueue(c, x, y, s, t);
}

int whb_imp_rhs(whb_ctx *c, int wi, int wpi, int lapi, int fi, int rhsi, int guessi, int first, double q0,
                double qh, double qd, double fs) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(w, wi);
    VEC_OR_FAIL(wp, wpi);
    VEC_OR_FAIL(lap, lapi);
    VEC_OR_FAIL(f, fi);
    VEC_OR_FAIL(rhs, rhsi);
    VEC_OR_FAIL(guess, guessi);
    ELEMWISE_LAUNCH(imp::rhs_kernel, owned(w, c), owned(wp, c), owned(lap, c), owned(f, c), owned(rhs, c),
                    owned(guess, c), first, q0, qh, qd, fs, owned_elems(c));
    return 0;
}

int whb_vec_xpay(whb_ctx *c, int xi, double a, int yi) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(x, xi);
    VEC_OR_FAIL(y, yi);
    ELEMWISE_LAUNCH(imp::xpay_kernel, owned(x, c), a, owned(y, c), owned_elems(c));
    return 0;
}

int whb_mg_setup(whb_ctx *c, int nlev, const int64_t *cells, const double *gamma, const double *diag,
                 const double *coarse_inv, int nu1, int nu2) {
    if (!c || !cells || !gamma || !diag || !coarse_inv) return fail(WHB_E_ARG, "NULL argument");
    if (c->ndim != 2 || c->plane_begin != 0 || c->plane_end != c->gshape[0])
        return fail(WHB_E_ARG, "multigrid needs a whole-grid 2D context");
    if (nlev < 1 || nu1 < 0 || nu2 < 0) return fail(WHB_E_ARG, "bad multigrid shape");
    if (cells[0] != c->gshape[0] - 1 || cells[1] != c->gshape[2] - 1)
        return fail(WHB_E_ARG, "level 0 must be the context grid");
    for (int l = 1; l < nlev; ++l)
        if (2 * cells[2 * l] != cells[2 * l - 2] || 2 * cells[2 * l + 1] != cells[2 * l - 1])
            return fail(WHB_E_ARG, "levels must halve the cell counts");
    WHB_TRY(set_dev(c));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    drop_cg_graphs(c);
    free_mg(c);
    c->mg = new MGData();
    MGData &M = *c->mg;
    M.nu1 = nu1;
    M.nu2 = nu2;
    M.lv.resize(nlev);
    auto fail_free = [&](int rc) { free_mg(c); return rc; };
    for (int l = 0; l < nlev; ++l) {
        MGLevelBuf &B = M.lv[l];
        B.lev.nx = (int)cells[2 * l];
        B.lev.ny = (int)cells[2 * l + 1];
        B.lev.gx = gamma[2 * l];
        B.lev.gy = gamma[2 * l + 1];
        B.lev.diag = diag[l];
        if (l == 0) {
            B.lev.rs = c->S0;  // 2D storage: one row per plane
            double *r = nullptr;
            int rc = alloc_field(c, &r);
            if (rc) return fail_free(rc);
            B.raw[2] = r - c->slack_front;  // freed as a raw allocation
            B.r = owned(r, c);
        } else {
            B.lev.rs = (B.lev.ny + 1 + 15) / 16 * 16;
            const size_t n = (size_t)(B.lev.nx + 1) * B.lev.rs;
            for (int q = 0; q < 3; ++q) {
                if (cudaMalloc(&B.raw[q], n * sizeof(double)) != cudaSuccess) return fail_free(fail(WHB_E_NOMEM, "mg level"));
                if (cudaMemsetAsync(B.raw[q], 0, n * sizeof(double), c->stream) != cudaSuccess)
                    return fail_free(fail(WHB_E_CUDA, "mg memset"));
            }
            B.u = B.raw[0];
            B.b = B.raw[1];
            B.r = B.raw[2];
        }
    }
    const imp::Lev &C = M.lv[nlev - 1].lev;
    const size_t nc = (size_t)(C.nx - 1) * (C.ny - 1);
    if (cudaMalloc(&M.ainv, nc * nc * sizeof(double)) != cudaSuccess) return fail_free(fail(WHB_E_NOMEM, "mg coarse"));
    if (cudaMemcpy(M.ainv, coarse_inv, nc * nc * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
        return fail_free(fail(WHB_E_CUDA, "mg coarse upload"));
    // single-CTA coarse sub-cycle: the deepest levels (>= 1, at least two of them) whose arrays
    // fit in 160 KB of shared memory together, with a small coarse system
    const char *cenv = getenv("WHB_MG_COARSE_CTA");
    if (!(cenv && std::string(cenv) == "0") && nc <= 1024) {
        size_t bytes = 0;
        int lc = -1;
        for (int l = nlev - 1; l >= 1; --l) {
            const imp::Lev &Lv = M.lv[l].lev;
            bytes += 2 * (size_t)(Lv.nx + 1) * (Lv.ny + 1) * sizeof(double);
            if (bytes > 160 * 1024 || nlev - l > imp::kMaxCoarseLevels) break;
            lc = l;
        }
        if (lc >= 1 && lc < nlev - 1) {
            M.lc = lc;
            M.cc.nlev = nlev - lc;
            M.cc.nu1 = nu1;
            M.cc.nu2 = nu2;
            M.cc.grs = M.lv[lc].lev.rs;
            M.cc_smem = 0;
            for (int l = lc; l < nlev; ++l) {
                imp::Lev Lv = M.lv[l].lev;
                Lv.rs = Lv.ny + 1;
                M.cc.lev[l - lc] = Lv;
                M.cc_smem += 2 * (size_t)(Lv.nx + 1) * (Lv.ny + 1) * sizeof(double);
            }
            if (cudaFuncSetAttribute(imp::coarse_cycle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)M.cc_smem) != cudaSuccess)
                M.lc = -1;
        }
    }
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
}

int whb_mg_vcycle(whb_ctx *c, int bi, int ui) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (!c->mg) return fail(WHB_E_STATE, "multigrid not set up (whb_mg_setup)");
    if (bi == ui) return fail(WHB_E_ARG, "whb_mg_vcycle needs distinct b and u");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(b, bi);
    VEC_OR_FAIL(u, ui);
    MGData &M = *c->mg;
    M.lv[0].b = owned(b, c);
    M.lv[0].u = owned(u, c);
    WHB_CUDA(cudaMemsetAsync(u - c->slack_front, 0,
                             (size_t)(c->slack_front + c->field_elems + c->slack_back) * sizeof(double), c->stream));
    if (!c->use_graphs) return mg_enqueue(c, 0);
    auto key = std::make_pair((const double *)b, (const double *)u);
    auto it = M.graphs.find(key);
    if (it == M.graphs.end()) {
        cudaGraph_t g;
        const int64_t l0 = c->launches;
        WHB_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        int rc = mg_enqueue(c, 0);
        cudaError_t e = cudaStreamEndCapture(c->stream, &g);
        if (rc) return rc;
        if (e != cudaSuccess) return fail(WHB_E_CUDA, std::string("capture: ") + cudaGetErrorString(e));
        cudaGraphExec_t ge;
        e = cudaGraphInstantiate(&ge, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return fail(WHB_E_CUDA, std::string("instantiate: ") + cudaGetErrorString(e));
        c->graph_kernels[std::make_tuple(-1, 0, (const void *)ge)] = c->launches - l0;
        c->launches = l0;
        it = M.graphs.emplace(key, ge).first;
    }
    WHB_CUDA(cudaGraphLaunch(it->second, c->stream));
    c->launches += c->graph_kernels[std::make_tuple(-1, 0, (const void *)it->second)];
    return 0;
}

int whb_tri_setup(whb_ctx *c, int n, const double *sub, const double *dp, const double *cp) {
    if (!c || !sub || !dp || !cp) return fail(WHB_E_ARG, "NULL argument");
    if (c->ndim != 1 || n != (int)c->gshape[2] - 2) return fail(WHB_E_ARG, "tridiagonal solve needs a 1D context with n = points - 2");
    WHB_TRY(set_dev(c));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    drop_cg_graphs(c);
    free_tri(c);
    c->tri = new TriData();
    TriData &T = *c->tri;
    T.n = n;
    const size_t b = (size_t)std::max(1, n) * sizeof(double);
    if (cudaMalloc(&T.sub, b) != cudaSuccess || cudaMalloc(&T.dp, b) != cudaSuccess ||
        cudaMalloc(&T.cp, b) != cudaSuccess || cudaMalloc(&T.y, b) != cudaSuccess) {
        free_tri(c);
        return fail(WHB_E_NOMEM, "tridiagonal factors");
    }
    if (n > 1) WHB_CUDA(cudaMemcpy(T.sub, sub, (n - 1) * sizeof(double), cudaMemcpyHostToDevice));
    WHB_CUDA(cudaMemcpy(T.dp, dp, n * sizeof(double), cudaMemcpyHostToDevice));
    if (n > 1) WHB_CUDA(cudaMemcpy(T.cp, cp, (n - 1) * sizeof(double), cudaMemcpyHostToDevice));
    return 0;
}

int whb_tri_solve(whb_ctx *c, int bi, int xi) {
    if (!c) return fail(WHB_E_ARG, "NULL argument");
    if (!c->tri) return fail(WHB_E_STATE, "tridiagonal factors not set (whb_tri_setup)");
    if (bi == xi) return fail(WHB_E_ARG, "whb_tri_solve needs distinct b and x");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(b, bi);
    VEC_OR_FAIL(x, xi);
    TriData &T = *c->tri;
    // x = scatter_interior(solve(interior_values(b))): boundary points of x are 0 (grid.py:548-556)
    WHB_CUDA(cudaMemsetAsync(owned(x, c), 0, (size_t)owned_elems(c) * sizeof(double), c->stream));
    imp::tri_solve_kernel<<<1, 32, 0, c->stream>>>(owned(b, c) + 1, owned(x, c) + 1, T.n, T.sub, T.dp, T.cp, T.y);
    c->launches++;
    WHB_CUDA(cudaGetLastError());
    return 0;
}

int whb_cg_begin(whb_ctx *c, int ri, int zi, int pi, int precond, double *rr) {
    if (!c || !rr) return fail(WHB_E_ARG, "NULL argument");
    if (precond < 0 || precond > 2) return fail(WHB_E_ARG, "precond must be 0, 1 or 2");
    if ((precond == 0) != (ri == zi)) return fail(WHB_E_ARG, "z is r exactly when there is no preconditioner");
    if (precond == 1 && !c->mg) return fail(WHB_E_STATE, "multigrid not set up");
    if (precond == 2 && !c->tri) return fail(WHB_E_STATE, "tridiagonal factors not set");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(r, ri);
    VEC_OR_FAIL(z, zi);
    VEC_OR_FAIL(p, pi);
    if (!c->d_cg) WHB_CUDA(cudaMalloc(&c->d_cg, imp::CG_NSC * sizeof(double)));
    WHB_TRY(precond_enqueue(c, r, z, precond));
    WHB_CUDA(cudaMemcpyAsync(p, z, (size_t)c->field_elems * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    WHB_TRY(cg_dot(c, r, z, 3));
    WHB_TRY(cg_dot(c, r, r, 1));
    WHB_CUDA(cudaMemcpyAsync(c->h_red, c->d_cg + imp::CG_RR, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    *rr = c->h_red[0];
    return 0;
}

int whb_cg_iterate(whb_ctx *c, int xi, int ri, int zi, int pi, int api, int tmpi, double s, int precond, double *pap,
                   double *rr) {
    if (!c || !pap || !rr) return fail(WHB_E_ARG, "NULL argument");
    if (!c->d_cg) return fail(WHB_E_STATE, "whb_cg_iterate before whb_cg_begin");
    if ((precond == 0) != (ri == zi)) return fail(WHB_E_ARG, "z is r exactly when there is no preconditioner");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(x, xi);
    VEC_OR_FAIL(r, ri);
    VEC_OR_FAIL(z, zi);
    VEC_OR_FAIL(p, pi);
    VEC_OR_FAIL(ap, api);
    double *t = nullptr;
    if (c->kern == 3) {
        VEC_OR_FAIL(tv, tmpi);
        t = tv;
    }
    auto enqueue = [&]() -> int {
        WHB_TRY(imp_apply_enqueue(c, p, ap, s, t));                     // Ap = A p
        WHB_TRY(cg_dot(c, p, ap, 0));                                   // pAp, alpha = rz / pAp
        imp::cg_update_kernel<<<kRedBlocks, kRedThreads, 0, c->stream>>>(owned(x, c), owned(r, c), owned(p, c),
                                                                         owned(ap, c), c->d_cg, owned_elems(c));
        c->launches++;
        WHB_TRY(cg_dot(c, r, r, 1));                                    // rnorm^2
        WHB_TRY(precond_enqueue(c, r, z, precond));                     // z = M r
        WHB_TRY(cg_dot(c, r, z, 2));                                    // rz_new, beta, rz = rz_new
        imp::cg_dir_kernel<<<kRedBlocks, kRedThreads, 0, c->stream>>>(owned(z, c), owned(p, c), c->d_cg,
                                                                      owned_elems(c));
        c->launches++;
        WHB_CUDA(cudaMemcpyAsync(c->h_red, c->d_cg, 4 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        WHB_CUDA(cudaGetLastError());
        return 0;
    };
    if (!c->use_graphs) {
        WHB_TRY(enqueue());
    } else {
        auto key = std::make_tuple(xi, ri, zi, pi, api, tmpi, precond, s);
        auto it = c->cg_graphs.find(key);
        if (it == c->cg_graphs.end()) {
            cudaGraph_t g;
            const int64_t l0 = c->launches;
            WHB_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
            int rc = enqueue();
            cudaError_t e = cudaStreamEndCapture(c->stream, &g);
            if (rc) return rc;
            if (e != cudaSuccess) return fail(WHB_E_CUDA, std::string("capture: ") + cudaGetErrorString(e));
            cudaGraphExec_t ge;
            e = cudaGraphInstantiate(&ge, g, 0);
            cudaGraphDestroy(g);
            if (e != cudaSuccess) return fail(WHB_E_CUDA, std::string("instantiate: ") + cudaGetErrorString(e));
            c->graph_kernels[std::make_tuple(-2, 0, (const void *)ge)] = c->launches - l0;
            c->launches = l0;
            it = c->cg_graphs.emplace(key, ge).first;
        }
        WHB_CUDA(cudaGraphLaunch(it->second, c->stream));
        c->launches += c->graph_kernels[std::make_tuple(-2, 0, (const void *)it->second)];
    }
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    *pap = c->h_red[imp::CG_PAP];
    *rr = c->h_red[imp::CG_RR];
    return 0;
}

int whb_vec_mgs(whb_ctx *c, int wi, int q_first, int count, int q_next, double *h_out) {
    if (!c || !h_out) return fail(WHB_E_ARG, "NULL argument");
    if (count < 1) return fail(WHB_E_ARG, "count must be >= 1");
    WHB_TRY(set_dev(c));
    VEC_OR_FAIL(w, wi);
    std::vector<double *> q(count);
    for (int j = 0; j < count; ++j) {
        q[j] = vec_ptr(c, q_first + j);
        if (!q[j]) return fail(WHB_E_ARG, "unknown basis vector id");
    }
    double *qn = nullptr;
    if (q_next >= 0) {
        qn = vec_ptr(c, q_next);
        if (!qn) return fail(WHB_E_ARG, "unknown vector id for the next basis vector");
    }
    if (count + 1 > c->mgs_cap) {
        cudaFree(c->d_mgs);
        if (c->h_mgs) cudaFreeHost(c->h_mgs);
        c->d_mgs = c->h_mgs = nullptr;
        c->mgs_cap = std::max(64, 2 * (count + 1));
        WHB_CUDA(cudaMalloc(&c->d_mgs, c->mgs_cap * sizeof(double)));
        WHB_CUDA(cudaMallocHost(&c->h_mgs, c->mgs_cap * sizeof(double)));
    }
    const long long n = owned_elems(c);
    for (int j = 0; j <= count; ++j) {
        // j < count: w -= h[j-1] q[j-1]; h[j] = q[j].w   j == count: w -= h[count-1] q[count-1]; h[count] = w.w
        const double *qp = j > 0 ? owned(q[j - 1], c) : nullptr;
        const double *qj = j < count ? owned(q[j], c) : nullptr;
        double *wo = owned(w, c);
        mgs_step_kernel<<<kRedBlocks, kRedThreads, 0, c->stream>>>(wo, qp, j > 0 ? c->d_mgs + (j - 1) : nullptr, qj,
                                                                   n, c->d_red);
        final_sum_kernel<<<1, 1024, 0, c->stream>>>(c->d_red, kRedBlocks, c->d_mgs + j);
        c->launches += 2;
    }
    if (qn) {
        mgs_normalise_kernel<<<kRedBlocks, kRedThreads, 0, c->stream>>>(owned(w, c), c->d_mgs + count, owned(qn, c), n);
        c->launches++;
    }
    WHB_CUDA(cudaGetLastError());
    WHB_CUDA(cudaMemcpyAsync(c->h_mgs, c->d_mgs, (count + 1) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    WHB_CUDA(cudaStreamSynchronize(c->stream));
    std::memcpy(h_out, c->h_mgs, (count + 1) * sizeof(double));
    return 0;
}

}  // extern "C"
