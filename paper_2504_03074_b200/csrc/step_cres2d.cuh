// Cluster-resident 2D solve for small grids (sm_100a): BASELINE config 1 (129^2) and any
// whole-grid 2D problem whose fields fit in the shared memory of one thread-block cluster.
//
// The multi-pass kernels stream every field through HBM once per pass; at 129^2 (16.6 K points)
// a pass is ~1 us of traffic but ~5-7 us of launch + pipeline fill, so config 1 ran at 8 Gpts/s.
// Here one cluster of CL CTAs (CL <= 16, one per SM) owns one problem for a whole launch:
//
//   * CTA r of the cluster owns the band of interior rows [rb, re) (CL near-equal bands).  Its
//     shared memory holds two time-level buffers (W^n and W^{n+1}/W^{n-1}, each with one halo
//     row above and below the band), f, acc, v and the per-step scalars (cos(w t^n),
//     (cos - alpha/2) sigma_n): every step of every iteration is computed from shared memory.
//   * Step n reads W^n from buffer n&1 and writes W^{n+1} over W^{n-1} in the other buffer (the
//     point's own W^{n-1} is read by the same thread just before).  A band's first and last rows
//     are also stored into the neighbouring CTAs' halo rows with st.shared::cluster (DSMEM);
//     one cluster barrier (arrive.release / wait.acquire) per step orders those stores before
//     the neighbours' next reads and every read of a buffer before its next overwrite.
//   * The last step forms v_new = ((2/Tbar) dt) acc, its squared difference to v (residual),
//     and writes v_new as W^0 of the next fixed-point iteration into the buffer that step filled;
//     the CTA partial sums are exchanged through DSMEM so every CTA forms the same total (same
//     order), and the convergence test (tol) is taken inside the kernel.  A whole fpi_solve of
//     K iterations is ONE launch; v leaves shared memory only at the end.
//
// Arithmetic: the same explicitly rounded operations in the same order as every other kernel
// (reference order), so the iterates are bitwise those of the reference.
// Boundary rows/columns are never written and stay exactly 0.
#pragma once

namespace cres {

constexpr int NT = 1024;  // threads per CTA (one CTA per SM)
constexpr int MAX_CL = 16;

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared::cta address -> the same offset in CTA `rank` of the cluster (shared::cluster window)
__device__ __forceinline__ uint32_t map_rank(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

__device__ __forceinline__ void st_remote(uint32_t addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

// Band of interior rows owned by CTA r: [1 + r*NR/CL, 1 + (r+1)*NR/CL), NR = n0 - 2.
__host__ __device__ __forceinline__ int band_begin(int r, int NR, int CL) { return 1 + (int)(((long long)r * NR) / CL); }

// Shared-memory layout (doubles): buf[0] | buf[1] ((R+2) x W each) | f (R x W, absent when
// ZF) | acc | v (R x W) | cos_f[Nmax] | acc_c[Nmax + 1] | partials[CL]
__host__ __device__ __forceinline__ size_t smem_doubles(int R, int W, bool zf, int nmax, int CL) {
    return (size_t)2 * (R + 2) * W + (size_t)(zf ? 2 : 3) * R * W + (size_t)(2 * nmax + 1) + CL;
}

struct Args {
    int CL;           // CTAs per cluster
    int R;            // max rows per band (buffer sizing)
    int W;            // shared row pitch (= n2)
    int nmax;         // max n_total over the launched members (scalar table sizing)
    int iters;        // fixed-point iterations (FPI mode), 1 otherwise
    double tol_sq;    // root_n <= 0: stop when resid^2 <= tol_sq (< 0: never)
    double tol, root_n;  // root_n > 0: stop when sqrt(resid^2) / root_n <= tol (< 0: never), driver.py:225-230
    double *hist;     // FPI: hist[(k0 + it) * nb + member idx] (nullptr: partials[0] for the reduction kernel)
    int k0, nb;
    int *done;        // FPI: iterations performed (written by member 0's cluster), may be nullptr
    int dbg;
};

template <int KIND, bool ZF, bool SQ>
__device__ __forceinline__ double cres_point(const Geom &g, const double *cur, int c, int W, double fv, double wpv,
                                             double h, double cosn) {
    return bulk::update_point<KIND, ZF, false, SQ>(g, cur[c - W], cur[c], cur[c + W], 0.0, 0.0, cur[c - 1],
                                                   cur[c + 1], fv, wpv, h, cosn);
}

template <bool ZF, bool SQ>
__global__ void __launch_bounds__(NT, 1)
    cres2d_kernel(Geom g, const Member *__restrict__ members, int member_off, Args a) {
    extern __shared__ __align__(16) double sm[];
    const Member m = members[member_off + blockIdx.y];
    const int CL = a.CL, W = a.W, n2 = g.n2;
    const int rank = (int)cta_rank();
    const int NR = g.i_hi - g.i_lo;  // interior rows (global rows 1 .. n0-2)
    const int rb = band_begin(rank, NR, CL), re = band_begin(rank + 1, NR, CL);
    const int nr = re - rb;
    const int nr_up = rank > 0 ? rb - band_begin(rank - 1, NR, CL) : 0;
    const bool has_up = rank > 0, has_dn = rank < CL - 1;
    const size_t BUF = (size_t)(a.R + 2) * W;
    double *buf0 = sm, *buf1 = sm + BUF;
    double *fs = buf1 + BUF;
    double *accs = fs + (ZF ? 0 : (size_t)a.R * W);
    double *vs = accs + (size_t)a.R * W;
    double *cosf = vs + (size_t)a.R * W;
    double *accc = cosf + a.nmax;
    double *part = accc + a.nmax + 1;
    const int N = m.n_total;
    const long long S0 = g.S0;
    const int GH0 = g.i_lo - 1;  // local plane of global row 0 (= ghost planes)

    // zero everything (boundary columns, halo rows at the global boundary), then load v (band +
    // the rows above/below it: W^0 halos), f and the scalar tables
    const size_t total = smem_doubles(a.R, W, ZF, a.nmax, CL);
    for (size_t i = threadIdx.x; i < total; i += NT) sm[i] = 0.0;
    __syncthreads();
    for (int t = threadIdx.x; t < (nr + 2) * n2; t += NT) {
        const int lr = t / n2, k = t - lr * n2;  // buffer row lr <-> global row rb - 1 + lr
        const double x = m.v[(long long)(GH0 + rb - 1 + lr) * S0 + k];
        buf0[lr * W + k] = x;
        if (lr >= 1 && lr <= nr) vs[(lr - 1) * W + k] = x;
    }
    if (!ZF)
        for (int t = threadIdx.x; t < nr * n2; t += NT) {
            const int lr = t / n2, k = t - lr * n2;
            fs[lr * W + k] = m.f[(long long)(GH0 + rb + lr) * S0 + k];
        }
    for (int t = threadIdx.x; t < N; t += NT) cosf[t] = m.cos_f[t];
    for (int t = threadIdx.x; t <= N; t += NT) accc[t] = m.acc_c[t];
    // remote halo rows: my first row lands in the upper neighbour's bottom halo row (nr_up + 1),
    // my last row in the lower neighbour's top halo row (0); per buffer
    uint32_t up0 = 0, up1 = 0, dn0 = 0, dn1 = 0;
    if (has_up) {
        up0 = map_rank(bulk::smem_u32(buf0 + (size_t)(nr_up + 1) * W), rank - 1);
        up1 = map_rank(bulk::smem_u32(buf1 + (size_t)(nr_up + 1) * W), rank - 1);
    }
    if (has_dn) {
        dn0 = map_rank(bulk::smem_u32(buf0), rank + 1);
        dn1 = map_rank(bulk::smem_u32(buf1), rank + 1);
    }
    const uint32_t part_local = bulk::smem_u32(part + rank);

    // thread -> (row group, column) map: TXc columns (warp multiple) x TY row groups
    const int ncol = n2 - 2;
    const int TXc = min(NT, (ncol + 31) / 32 * 32);
    const int TY = NT / TXc;
    const int tx = threadIdx.x % TXc, ty = threadIdx.x / TXc;
    const bool active = ty < TY;

    const bool fpi = m.out_mode == WHB_OUT_FPI;
    int p = 0;  // buffer holding W^0 of the current iteration
    int it = 0;
    cluster_sync();  // shared memory initialised cluster-wide before any remote store
    const double acc0 = accc[0], osc = m.out_scale;  // (the table is filled before the barrier)
    for (; it < a.iters; ++it) {
        double rsum = 0.0;
        for (int s = 0; s < N; ++s) {
            const int bc = (s + p) & 1;
            const double *cur = bc ? buf1 : buf0;
            double *nxt = bc ? buf0 : buf1;
            const uint32_t upb = bc ? up0 : up1, dnb = bc ? dn0 : dn1;  // remote halos of nxt
            const double h = s == 0 ? m.half_dt2 : m.dt2;
            const double cosn = s == 0 ? 1.0 : cosf[s];
            const double accn = accc[s + 1];
            if (active) {
                for (int lr = ty; lr < nr; lr += TY) {
                    for (int k = 1 + tx; k < n2 - 1; k += TXc) {
                        const int c = (lr + 1) * W + k;  // buffer index (row lr of the band)
                        const int o = lr * W + k;        // band index (f, acc, v)
                        const double fv = ZF ? 0.0 : fs[o];
                        double wn, out = 0.0;
                        bool store = true;
                        if (s == 0) {
                            wn = cres_point<K_FIRST, ZF, SQ>(g, cur, c, W, fv, 0.0, h, cosn);
                            const double ac = whb_add(whb_mul(acc0, cur[c]), whb_mul(accn, wn));
                            if (s == N - 1) out = whb_mul(osc, ac);
                            else accs[o] = ac;
                        } else {
                            wn = cres_point<K_MID, ZF, SQ>(g, cur, c, W, fv, nxt[c], h, cosn);
                            const double ac = whb_add(accs[o], whb_mul(accn, wn));
                            if (s == N - 1) out = whb_mul(osc, ac);
                            else accs[o] = ac;
                        }
                        if (s == N - 1) {
                            const double vo = vs[o];
                            if (fpi) {
                                const double d = out - vo;
                                rsum += d * d;
                                vs[o] = out;
                                wn = out;  // W^0 of the next iteration
                            } else {
                                double *dst = m.dst + (long long)(GH0 + rb + lr) * S0 + k;
                                *dst = (m.out_mode == WHB_OUT_AV) ? whb_sub(vo, out) : out;
                                store = false;
                            }
                        }
                        if (store) {
                            nxt[c] = wn;
                            if (!(a.dbg & 8)) {
                                if (lr == 0 && has_up) st_remote(upb + 8u * k, wn);
                                if (lr == nr - 1 && has_dn) st_remote(dnb + 8u * k, wn);
                            }
                        }
                    }
                }
            }
            if (s == N - 1 && fpi) {
                // CTA partial -> slot `rank` of every CTA's partial table (ordered by the barrier below)
                const double b = block_sum(rsum);
                if (threadIdx.x == 0)
                    for (int q = 0; q < CL; ++q) st_remote(map_rank(part_local, q), b);
            }
            if (a.dbg & 2) __syncthreads();
            cluster_sync();
            if (a.dbg & 1) __syncthreads();
            if (a.dbg & 4) cluster_sync();
        }
        p ^= (N & 1);  // the last step wrote W^0 of the next iteration into buffer (N + p) & 1
        if (!fpi) {
            ++it;
            break;
        }
        double r2 = 0.0;
        for (int q = 0; q < CL; ++q) r2 += part[q];  // same order in every CTA
        if (rank == 0 && threadIdx.x == 0) {
            if (a.hist) a.hist[(long long)(a.k0 + it) * a.nb + m.idx] = r2;
            else m.partials[0] = r2;
        }
        const bool stop = a.root_n > 0.0 ? (a.tol >= 0.0 && __ddiv_rn(__dsqrt_rn(r2), a.root_n) <= a.tol)
                                         : (a.tol_sq >= 0.0 && r2 <= a.tol_sq);
        if (stop) {
            ++it;
            break;
        }
    }
    // the iterate (FPI) back to HBM
    if (fpi)
        for (int t = threadIdx.x; t < nr * n2; t += NT) {
            const int lr = t / n2, k = t - lr * n2;
            m.v[(long long)(GH0 + rb + lr) * S0 + k] = vs[lr * W + k];
        }
    if (a.done && blockIdx.y == 0 && rank == 0 && threadIdx.x == 0) *a.done = it;
    cluster_sync();  // no CTA exits while a neighbour may still address its shared memory
}

}  // namespace cres
