// 3D two-step kernel, one row of work per warp per phase (sm_100a).
//
// Same algorithm as tb2_kernel (two leapfrog steps per pass, TMA tensor boxes,
// W^{s+1} of the extended tile in a 3-plane shared-memory ring), re-tiled so
// the work is perfectly balanced: the CTA's output tile is BY rows x 62
// columns starting at an odd column k0, so its extended tile (one extra cell
// around it) is (BY+2) rows x 64 columns = 32 lane pairs per row, aligned to
// even columns.  CTA = BY+2 warps: in phase 1 warp w computes W^{s+1} on
// extended row w (all 32 lanes busy), in phase 2 warps 0..BY-1 compute
// W^{s+2} on the output rows (their first/last lane pair straddles the tile
// edge; only in-tile points are written).  The previous layout (64-column
// tiles) left the extended ring to 4 of 16 warps, a 2-units-vs-1 critical
// path in phase 1.
//
// Boxes (all starting at even columns, so every 16-byte smem access is aligned):
//   W^s     (BY+4) x 68 at (k0-3, j0-2)     W^{s-1}, f  (BY+2) x 64 at (k0-1, j0-1)
//   acc      BY    x 64 at (k0-1, j0)        E ring      3 x (BY+2) x 68 (col c at c-(k0-3))
#pragma once

namespace tb2r {

using bulk::fence_proxy_async;
using bulk::mbar_expect_tx;
using bulk::mbar_init;
using bulk::mbar_wait;
using bulk::tma_load_3d;
using bulk::update_point;

constexpr int pad16(int x) { return (x + 15) / 16 * 16; }

template <int BY>
struct Lay {
    static constexpr int TX = 62;                      // output columns per CTA
    static constexpr int WW = 68;                      // W^s box / E ring row width
    static constexpr int PW = 64;                      // prev / f / acc box row width
    static constexpr int W_EL = pad16((BY + 4) * WW);
    static constexpr int P_EL = pad16((BY + 2) * PW);
    static constexpr int A_EL = pad16(BY * PW);
    static constexpr int STAGE = W_EL + 2 * P_EL + A_EL;
    static constexpr int E_EL = pad16((BY + 2) * WW);
    static constexpr int THREADS = 32 * (BY + 2);
};

template <int BY, int ST>
constexpr size_t smem_bytes() {
    using L = Lay<BY>;
    return (size_t)(ST * L::STAGE + 3 * L::E_EL) * sizeof(double) + ST * sizeof(uint64_t);
}

template <int BY, int ST, int K1, int K2, bool ZF>
__global__ void __launch_bounds__(Lay<BY>::THREADS)
    tb2r_kernel(Geom g, const Member *__restrict__ members, int member_off, int s, int i_begin, int i_end,
                int chunk_len, int JT, int part_off, const __grid_constant__ CUtensorMap tm_w,
                const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_f,
                const __grid_constant__ CUtensorMap tm_a) {
    using L = Lay<BY>;
    static_assert(ST >= 4, "3 live planes + 1 in flight");
    extern __shared__ __align__(128) double smem[];
    double *ering = smem + (size_t)ST * L::STAGE;
    uint64_t *bars = reinterpret_cast<uint64_t *>(ering + 3 * L::E_EL);

    const Member m = members[member_off + blockIdx.z];
    const int tid = threadIdx.x;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const int lane = tid & 31;
    const int jt = blockIdx.y % JT;
    const int ch = blockIdx.y / JT;
    const int k0 = 1 + blockIdx.x * L::TX;  // odd: first output column of the tile
    const int j0 = jt * BY;
    const int i0 = i_begin + ch * chunk_len;
    const int i1 = min(i_end, i0 + chunk_len);
    if (i0 >= i1) {
        if (K2 == K_LAST && m.out_mode == WHB_OUT_FPI && tid == 0)
            m.partials[part_off + blockIdx.y * gridDim.x + blockIdx.x] = 0.0;
        return;
    }
    double *w1g = level_ptr(m, s + 1);
    double *w2g = level_ptr(m, s + 2);
    const double h1 = (K1 == K_FIRST) ? m.half_dt2 : m.dt2;
    const double cos1 = (K1 == K_FIRST) ? 1.0 : m.cos_f[s];
    const double cos2 = m.cos_f[s + 1];
    const double h2 = m.dt2;
    const double acc0 = m.acc_c[0];
    const double c1 = m.acc_c[s + 1];
    const double c2 = m.acc_c[s + 2];
    const long long S0 = g.S0;
    const int P = g.P;

    constexpr bool LOAD_P = (K1 != K_FIRST);
    constexpr bool LOAD_A = (K1 != K_FIRST);
    constexpr uint32_t W_BYTES = (BY + 4) * L::WW * 8;
    constexpr uint32_t P_BYTES = (BY + 2) * L::PW * 8;
    constexpr uint32_t A_BYTES = BY * L::PW * 8;
    constexpr uint32_t stage_bytes = W_BYTES + (LOAD_P ? P_BYTES : 0) + (ZF ? 0 : P_BYTES) + (LOAD_A ? A_BYTES : 0);
    const int n_st = i1 - i0 + 4;  // planes i0-2 .. i1+1

    auto issue = [&](int t) {
        const int slot = t % ST;
        double *st = smem + (size_t)slot * L::STAGE;
        double *sp = st + L::W_EL, *sf = sp + L::P_EL, *sa = sf + L::P_EL;
        uint64_t *bar = bars + slot;
        const int plane = i0 - 2 + t;
        mbar_expect_tx(bar, stage_bytes);
        tma_load_3d(st, &tm_w, k0 - 3, j0 - 2, plane, bar);
        if (LOAD_P) tma_load_3d(sp, &tm_p, k0 - 1, j0 - 1, plane, bar);
        if (!ZF) tma_load_3d(sf, &tm_f, k0 - 1, j0 - 1, plane, bar);
        if (LOAD_A) tma_load_3d(sa, &tm_a, k0 - 1, j0, plane, bar);
    };

    if (tid == 0) {
        for (int t = 0; t < ST; ++t) mbar_init(bars + t, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const int pro = min(n_st, ST);
        for (int t = 0; t < pro; ++t) issue(t);
    }
    __syncthreads();

    // phase-1 row (extended row `warp`, y = j0 - 1 + warp) and phase-2 row (output row `warp`)
    const int cl = 2 * lane;                 // column pair offset: global columns k0-1+cl, k0+cl
    const int kx = k0 - 1 + cl;              // even global column of the pair
    const bool xin0 = kx >= 1 && kx < g.n2 - 1;
    const bool xin1 = kx + 1 >= 1 && kx + 1 < g.n2 - 1;
    const int ey = warp;                     // extended row index (0 .. BY+1)
    const int jy = j0 - 1 + ey;
    const bool y1in = jy >= g.j_lo && jy < g.j_hi;
    const bool p2 = warp < BY;               // phase-2 worker
    const int jo = j0 + warp;                // output row
    const bool orow_ok = p2 && jo >= g.j_lo && jo < g.j_hi;
    // in-tile output columns: [k0, k0+62) -> the pair's first point is out of tile for lane 0,
    // the second for lane 31
    const bool ok0 = orow_ok && xin0 && lane > 0;
    const bool ok1 = orow_ok && xin1 && lane < 31 && kx + 1 < k0 + L::TX;
    double rsum = 0.0;
    const bool want_v = (K2 == K_LAST) && m.out_mode != WHB_OUT_PLAIN && p2 && (ok0 || ok1);
    const long long pbase = (long long)jo * P + kx;
    double2 vcur = make_double2(0.0, 0.0);

    for (int i = i0 - 1; i <= i1; ++i) {
        const int t = i - i0 + 2;
        const double2 vnext = (want_v && i >= i0 && i < i1)
                                  ? *reinterpret_cast<const double2 *>(m.v + (long long)i * S0 + pbase)
                                  : make_double2(0.0, 0.0);
        if (i > i0 - 1) {
            __syncthreads();
            if (tid == 0) {
                const int tn = t - 2 + ST;
                if (tn < n_st) {
                    fence_proxy_async();
                    issue(tn);
                }
            }
        } else {
            mbar_wait(bars + ((t - 1) % ST), ((t - 1) / ST) & 1);
            mbar_wait(bars + (t % ST), (t / ST) & 1);
        }
        mbar_wait(bars + ((t + 1) % ST), ((t + 1) / ST) & 1);
        const double *sm_m = smem + (size_t)((t - 1) % ST) * L::STAGE;
        const double *sm_c = smem + (size_t)(t % ST) * L::STAGE;
        const double *sm_p = smem + (size_t)((t + 1) % ST) * L::STAGE;
        double *E = ering + (size_t)(i % 3) * L::E_EL;

        // ---- phase 1: W^{s+1}(plane i) on extended row ey (W box row ey+1, P/F row ey)
        {
            const int rw = ey + 1;  // W^s box row of jy (box starts at j0-2)
            const int cw = cl + 2;  // W^s box column of kx (box starts at k0-3)
            const double2 wc = *reinterpret_cast<const double2 *>(sm_c + rw * L::WW + cw);
            const double2 wm = *reinterpret_cast<const double2 *>(sm_m + rw * L::WW + cw);
            const double2 wp = *reinterpret_cast<const double2 *>(sm_p + rw * L::WW + cw);
            const double2 yl = *reinterpret_cast<const double2 *>(sm_c + (rw - 1) * L::WW + cw);
            const double2 yh = *reinterpret_cast<const double2 *>(sm_c + (rw + 1) * L::WW + cw);
            const double xl = sm_c[rw * L::WW + cw - 1];
            const double xh = sm_c[rw * L::WW + cw + 2];
            const double *P_ = sm_c + L::W_EL;
            const double *F_ = P_ + L::P_EL;
            double2 fv = make_double2(0.0, 0.0), pv = make_double2(0.0, 0.0);
            if (!ZF) fv = *reinterpret_cast<const double2 *>(F_ + ey * L::PW + cl);
            if (LOAD_P) pv = *reinterpret_cast<const double2 *>(P_ + ey * L::PW + cl);
            const double a = update_point<K1, ZF, true>(g, wm.x, wc.x, wp.x, yl.x, yh.x, xl, wc.y, fv.x, pv.x, h1, cos1);
            const double b = update_point<K1, ZF, true>(g, wm.y, wc.y, wp.y, yl.y, yh.y, wc.x, xh, fv.y, pv.y, h1, cos1);
            const bool pin = (i >= g.i_lo) && (i < g.i_hi) && y1in;
            *reinterpret_cast<double2 *>(E + ey * L::WW + cw) = make_double2((pin && xin0) ? a : 0.0,
                                                                             (pin && xin1) ? b : 0.0);
        }
        __syncthreads();

        // ---- phase 2: W^{s+2}(plane i-1) on output row warp (warps 0..BY-1)
        const int ip = i - 1;
        if (ip >= i0 && p2) {
            const double *Em = ering + (size_t)((ip + 2) % 3) * L::E_EL;
            const double *Ec = ering + (size_t)(ip % 3) * L::E_EL;
            const double *Ep = E;
            const double *st_c = sm_m;  // stage of plane ip
            const double *F_ = st_c + L::W_EL + L::P_EL;
            const double *A_ = F_ + L::P_EL;
            const int re = warp + 1;    // E row of output row `warp`
            const int cw = cl + 2;
            const double2 e_c = *reinterpret_cast<const double2 *>(Ec + re * L::WW + cw);
            const double2 e_m = *reinterpret_cast<const double2 *>(Em + re * L::WW + cw);
            const double2 e_p = *reinterpret_cast<const double2 *>(Ep + re * L::WW + cw);
            const double2 e_yl = *reinterpret_cast<const double2 *>(Ec + (re - 1) * L::WW + cw);
            const double2 e_yh = *reinterpret_cast<const double2 *>(Ec + (re + 1) * L::WW + cw);
            const double e_xl = Ec[re * L::WW + cw - 1];
            const double e_xh = Ec[re * L::WW + cw + 2];
            const double2 w0 = *reinterpret_cast<const double2 *>(st_c + (warp + 2) * L::WW + cw);
            const double2 f2 = ZF ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2 *>(F_ + re * L::PW + cl);
            const double n0 = update_point<K_MID, ZF, true>(g, e_m.x, e_c.x, e_p.x, e_yl.x, e_yh.x, e_xl, e_c.y, f2.x,
                                                           w0.x, h2, cos2);
            const double n1 = update_point<K_MID, ZF, true>(g, e_m.y, e_c.y, e_p.y, e_yl.y, e_yh.y, e_c.x, e_xh, f2.y,
                                                           w0.y, h2, cos2);
            double a0, a1;
            if (K1 == K_FIRST) {
                a0 = whb_add(whb_add(whb_mul(acc0, w0.x), whb_mul(c1, e_c.x)), whb_mul(c2, n0));
                a1 = whb_add(whb_add(whb_mul(acc0, w0.y), whb_mul(c1, e_c.y)), whb_mul(c2, n1));
            } else {
                const double2 ao = *reinterpret_cast<const double2 *>(A_ + warp * L::PW + cl);
                a0 = whb_add(whb_add(ao.x, whb_mul(c1, e_c.x)), whb_mul(c2, n0));
                a1 = whb_add(whb_add(ao.y, whb_mul(c1, e_c.y)), whb_mul(c2, n1));
            }
            const long long p = (long long)ip * S0 + (long long)jo * P + kx;
            if (K2 == K_MID) {
                if (ok0 && ok1) {
                    *reinterpret_cast<double2 *>(w1g + p) = e_c;
                    *reinterpret_cast<double2 *>(w2g + p) = make_double2(n0, n1);
                    *reinterpret_cast<double2 *>(m.acc + p) = make_double2(a0, a1);
                } else {
                    if (ok0) { w1g[p] = e_c.x; w2g[p] = n0; m.acc[p] = a0; }
                    if (ok1) { w1g[p + 1] = e_c.y; w2g[p + 1] = n1; m.acc[p + 1] = a1; }
                }
            } else {
                const double o0 = whb_mul(m.out_scale, a0);
                const double o1 = whb_mul(m.out_scale, a1);
                if (m.out_mode == WHB_OUT_FPI) {
                    if (ok0) { const double d = o0 - vcur.x; rsum += d * d; m.v[p] = o0; }
                    if (ok1) { const double d = o1 - vcur.y; rsum += d * d; m.v[p + 1] = o1; }
                } else if (m.out_mode == WHB_OUT_AV) {
                    if (ok0) m.dst[p] = whb_sub(vcur.x, o0);
                    if (ok1) m.dst[p + 1] = whb_sub(vcur.y, o1);
                } else {
                    if (ok0) m.dst[p] = o0;
                    if (ok1) m.dst[p + 1] = o1;
                }
            }
        }
        vcur = vnext;
    }
    if (K2 == K_LAST && m.out_mode == WHB_OUT_FPI) {
        const double tsum = block_sum(rsum);
        if (tid == 0) m.partials[part_off + blockIdx.y * gridDim.x + blockIdx.x] = tsum;
    }
}

}  // namespace tb2r
