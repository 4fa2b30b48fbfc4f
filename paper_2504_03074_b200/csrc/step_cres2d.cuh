// Cluster-resident 2D solve for small grids (sm_100a): BASELINE config 1 (129^2) and any
// whole-grid 2D problem whose fields fit in the shared memory of one thread-block cluster.
//
// The multi-pass kernels stream every field through HBM once per pass; at 129^2 (16.6 K points)
// a pass is ~1 us of traffic but ~5-7 us of launch + pipeline fill, so config 1 ran at 8 Gpts/s.
// Here one cluster of CL CTAs (CL <= 16, one per SM) owns one problem for a whole launch:
//
//   * CTA r of the cluster owns the band of interior rows [rb, re) (CL near-equal bands); each
//     thread owns up to PPT of its points and keeps their f, acc, v, W^n and W^{n-1} in
//     registers.  Shared memory holds two time-level buffers (each with one halo row above and
//     below the band) through which neighbours read W^n, and the per-step scalars (cos(w t^n),
//     (cos - alpha/2) sigma_n): every step of every iteration runs from registers + shared memory.
//   * Step n reads the 4 neighbours' W^n from buffer n&1 and publishes the point's W^{n+1} in the
//     other buffer (over W^{n-1}, which nobody reads any more).  A band's first and last rows
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

#ifndef WHB_CRES_NT
#define WHB_CRES_NT 512
#endif
constexpr int NT = WHB_CRES_NT;  // threads per CTA (one CTA per SM)
constexpr int MAX_PPT = 8;  // band points per thread (registers)
constexpr int MAX_CL = 16;

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Per-step barrier: shared-memory writes of this CTA are ordered by bar.sync; only the threads
// that stored into a neighbour's shared memory (DSMEM) fence at cluster scope before a relaxed
// cluster arrival (WHB_CRES_RELAXED variant; the default is the release/acquire cluster barrier).
__device__ __forceinline__ void step_sync(bool remote) {
#ifdef WHB_CRES_RELAXED
    if (remote) asm volatile("fence.acq_rel.cluster;" ::: "memory");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
#else
    (void)remote;
    cluster_sync();
#endif
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

// Neighbour-only step synchronisation (WHB_CRES_NBSYNC variant): an mbarrier per level buffer
// counts the neighbours' "my edge rows of this buffer are stored, and I finished reading the
// other buffer" arrivals (remote arrive with release at cluster scope after the CTA barrier).
__device__ __forceinline__ void mbar_remote_arrive(uint32_t remote_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_addr) : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster(uint32_t addr, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WHB_CW%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WHB_CW%=;\n}" ::"r"(addr),
        "r"(parity)
        : "memory");
}

// Band of interior rows owned by CTA r: [1 + r*NR/CL, 1 + (r+1)*NR/CL), NR = n0 - 2.
__host__ __device__ __forceinline__ int band_begin(int r, int NR, int CL) { return 1 + (int)(((long long)r * NR) / CL); }

// Shared-memory layout (doubles): buf[0] | buf[1] ((R+2) x W each) | cos_f[Nmax] |
// acc_c[Nmax + 1] | partials[CL].  f, acc, v and the point's own W^n, W^{n-1} live in registers.
__host__ __device__ __forceinline__ size_t smem_doubles(int R, int W, int nmax, int CL) {
    return (size_t)2 * (R + 2) * W + (size_t)(2 * nmax + 1) + CL + 2;  // + 2 mbarriers
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
};

// GM: geometry mode (wf2d.cuh): 1 = square cells, 2 = square cells and c^2 == 1
template <bool ZF, int GM, int PPT>
__global__ void __launch_bounds__(NT, 1)
    cres2d_kernel(Geom g, const Member *__restrict__ members, int member_off, Args a) {
    constexpr bool SQ = GM >= 1;
    constexpr int C2M = GM == 2 ? 0 : -1;
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
    double *cosf = buf1 + BUF;
    double *accc = cosf + a.nmax;
    double *part = accc + a.nmax + 1;
    uint64_t *nbar = reinterpret_cast<uint64_t *>(part + CL);  // per level buffer (NBSYNC variant)
    const int N = m.n_total;
    const long long S0 = g.S0;
    const int GH0 = g.i_lo - 1;  // local plane of global row 0 (= ghost planes)

    // zero the two level buffers (boundary columns, halo rows at the global boundary), then
    // W^0 = v on the band and the rows above/below it, and the scalar tables
    const size_t total = smem_doubles(a.R, W, a.nmax, CL);
    for (size_t i = threadIdx.x; i < total; i += NT) sm[i] = 0.0;
    __syncthreads();
#ifdef WHB_CRES_NBSYNC
    if (threadIdx.x == 0) {
        const uint32_t nn = (rank > 0 ? 1u : 0u) + (rank < CL - 1 ? 1u : 0u);
        bulk::mbar_init(nbar, nn > 0 ? nn : 1u);
        bulk::mbar_init(nbar + 1, nn > 0 ? nn : 1u);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t nphase[2] = {0u, 0u};
    const uint32_t nbar_local = bulk::smem_u32(nbar);
    const uint32_t nbar_up = rank > 0 ? map_rank(nbar_local, rank - 1) : 0u;
    const uint32_t nbar_dn = rank < CL - 1 ? map_rank(nbar_local, rank + 1) : 0u;
#endif
    for (int t = threadIdx.x; t < (nr + 2) * n2; t += NT) {
        const int lr = t / n2, k = t - lr * n2;  // buffer row lr <-> global row rb - 1 + lr
        buf0[lr * W + k] = m.v[(long long)(GH0 + rb - 1 + lr) * S0 + k];
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

    // the thread's points (band-interior point q = threadIdx.x + i * NT, row-major over nr x (n2-2)):
    // shared index, global offset, halo duties, and the point's own state in registers
    const int ncol = n2 - 2;
    const int npts = nr * ncol;
    int cidx[PPT], kidx[PPT];
    int goff[PPT];  // < 2^31: the grid fits in one cluster's shared memory
    bool ok[PPT], pu[PPT], pd[PPT];
    double wc[PPT], wp[PPT], fv[PPT], ac[PPT], vv[PPT];
#pragma unroll
    for (int i = 0; i < PPT; ++i) {
        const int q = threadIdx.x + i * NT;
        ok[i] = q < npts;
        const int lr = ok[i] ? q / ncol : 0;
        const int k = ok[i] ? 1 + (q - lr * ncol) : 1;
        cidx[i] = (lr + 1) * W + k;
        kidx[i] = k;
        goff[i] = (int)((long long)(GH0 + rb + lr) * S0 + k);
        pu[i] = ok[i] && lr == 0 && has_up;
        pd[i] = ok[i] && lr == nr - 1 && has_dn;
        vv[i] = ok[i] ? m.v[goff[i]] : 0.0;
        fv[i] = (ok[i] && !ZF) ? m.f[goff[i]] : 0.0;
        wc[i] = vv[i];
        wp[i] = 0.0;
        ac[i] = 0.0;
    }

    bool has_remote = false;
#pragma unroll
    for (int i = 0; i < PPT; ++i) has_remote = has_remote || pu[i] || pd[i];
    const bool fpi = m.out_mode == WHB_OUT_FPI;
    int p = 0;  // buffer holding W^0 of the current iteration
    int it = 0;
    cluster_sync();  // shared memory initialised cluster-wide before any read or remote store
    const double acc0 = accc[0], osc = m.out_scale;  // (the table is filled before the barrier)
    for (; it < a.iters; ++it) {
        double rsum = 0.0;
        for (int s = 0; s < N; ++s) {
            const int bc = (s + p) & 1;
            const double *cur = bc ? buf1 : buf0;
            double *nxt = bc ? buf0 : buf1;
            const uint32_t upb = bc ? up0 : up1, dnb = bc ? dn0 : dn1;  // remote halos of nxt
            const double accn = accc[s + 1];
            const bool last = s == N - 1;
#pragma unroll
            for (int i = 0; i < PPT; ++i) {
                if (!ok[i]) continue;
                const int c = cidx[i];
                double wn;
                if (s == 0) {
                    wn = bulk::update_point<K_FIRST, ZF, false, SQ, C2M>(g, cur[c - W], wc[i], cur[c + W], 0.0, 0.0,
                                                                  cur[c - 1], cur[c + 1], fv[i], 0.0, m.half_dt2, 1.0);
                    ac[i] = whb_add(whb_mul(acc0, wc[i]), whb_mul(accn, wn));
                } else {
                    wn = bulk::update_point<K_MID, ZF, false, SQ, C2M>(g, cur[c - W], wc[i], cur[c + W], 0.0, 0.0,
                                                                cur[c - 1], cur[c + 1], fv[i], wp[i], m.dt2, cosf[s]);
                    ac[i] = whb_add(ac[i], whb_mul(accn, wn));
                }
                wp[i] = wc[i];
                wc[i] = wn;
                if (last) {
                    const double out = whb_mul(osc, ac[i]);
                    if (fpi) {
                        const double d = out - vv[i];
                        rsum += d * d;
                        vv[i] = out;
                        wc[i] = out;  // W^0 of the next iteration
                    } else {
                        m.dst[goff[i]] = (m.out_mode == WHB_OUT_AV) ? whb_sub(vv[i], out) : out;
                        continue;
                    }
                }
                nxt[c] = wc[i];
                if (pu[i]) st_remote(upb + 8u * kidx[i], wc[i]);
                if (pd[i]) st_remote(dnb + 8u * kidx[i], wc[i]);
            }
            if (last && fpi) {
                // CTA partial -> slot `rank` of every CTA's partial table (ordered by the barrier below)
                const double b = block_sum(rsum);
                if (threadIdx.x == 0)
                    for (int q = 0; q < CL; ++q) st_remote(map_rank(part_local, q), b);
            }
#ifdef WHB_CRES_NBSYNC
            if (last) {
                cluster_sync();  // the residual partials: once per fixed-point iteration, whole cluster
            } else {
                __syncthreads();
                const int bn = bc ^ 1;  // buffer this step filled
                if (threadIdx.x == 0) {
                    if (has_up) mbar_remote_arrive(nbar_up + 8u * bn);
                    if (has_dn) mbar_remote_arrive(nbar_dn + 8u * bn);
                }
                if (has_up || has_dn) {
                    mbar_wait_cluster(nbar_local + 8u * bn, nphase[bn] & 1u);
                    nphase[bn]++;
                }
            }
#else
            step_sync(has_remote || (last && fpi && threadIdx.x == 0));
#endif
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
    if (fpi) {  // the iterate back to HBM
#pragma unroll
        for (int i = 0; i < PPT; ++i)
            if (ok[i]) m.v[goff[i]] = vv[i];
    }
    if (a.done && blockIdx.y == 0 && rank == 0 && threadIdx.x == 0) *a.done = it;
    cluster_sync();  // no CTA exits while a neighbour may still address its shared memory
}

}  // namespace cres
