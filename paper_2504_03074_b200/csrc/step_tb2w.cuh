// 3D two-step kernel, warp-specialised (sm_100a).
//
// Same arithmetic as tb2_kernel (steps s and s+1 fused; W^{s+1} on the tile
// extended by one cell, then W^{s+2} on the tile), but the two phases run in
// different warp groups that never meet at a CTA-wide barrier:
//
//   warp 30      producer: TMA tensor boxes of W^s, W^{s-1}, f, acc per plane
//                into a 5-stage ring ("full" mbarriers with tx counts; a stage
//                is refilled when all 30 compute warps arrived on "empty")
//   warps 0-15   group A: W^{s+1}(plane i) on extended row w (16 rows x 64
//                columns = 32 lane pairs) -> 4-plane ring E (E_full arrivals)
//   warps 16-29  group B: W^{s+2}(plane j) on output row w-16 from E planes
//                j-1, j, j+1 (E_empty arrivals release a slot to group A)
//
// so group A runs up to three planes ahead of group B and both overlap the
// TMA traffic.  Tile: BY = 14 output rows x 62 output columns from an odd
// column k0 (the extended tile is then exactly 32 even-aligned pairs wide).
#pragma once

namespace tb2w {

using bulk::mbar_expect_tx;
using bulk::mbar_init;
using bulk::mbar_wait;
using bulk::smem_u32;
using bulk::tma_load_3d;
using bulk::update_point;

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

constexpr int pad16(int x) { return (x + 15) / 16 * 16; }

template <int BY>
struct Lay {
    static constexpr int TX = 62, WW = 68, PW = 64;
    static constexpr int ER = BY + 2;                  // extended rows = group-A warps
    static constexpr int W_EL = pad16((BY + 4) * WW);
    static constexpr int P_EL = pad16(ER * PW);
    static constexpr int A_EL = pad16(BY * PW);
    static constexpr int STAGE = W_EL + 2 * P_EL + A_EL;
    static constexpr int E_EL = pad16(ER * WW);
    static constexpr int NA = ER, NB = BY;              // warps per group
    static constexpr int THREADS = 32 * (NA + NB + 1);
};

template <int BY, int ST>
constexpr size_t smem_bytes() {
    using L = Lay<BY>;
    return (size_t)(ST * L::STAGE + 4 * L::E_EL) * sizeof(double) + (2 * ST + 8) * sizeof(uint64_t);
}

template <int BY, int ST, int K1, int K2, bool ZF>
__global__ void __launch_bounds__(Lay<BY>::THREADS)
    tb2w_kernel(Geom g, const Member *__restrict__ members, int member_off, int s, int i_begin, int i_end,
                int chunk_len, int JT, int part_off, const __grid_constant__ CUtensorMap tm_w,
                const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_f,
                const __grid_constant__ CUtensorMap tm_a) {
    using L = Lay<BY>;
    static_assert(ST >= 5, "group A holds 3 planes, group B one more, plus one in flight");
    extern __shared__ __align__(128) double smem[];
    double *ering = smem + (size_t)ST * L::STAGE;
    uint64_t *full = reinterpret_cast<uint64_t *>(ering + 4 * L::E_EL);
    uint64_t *empty = full + ST;
    uint64_t *e_full = empty + ST;
    uint64_t *e_empty = e_full + 4;

    const Member m = members[member_off + blockIdx.z];
    const int tid = threadIdx.x;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
    const int lane = tid & 31;
    const int jt = blockIdx.y % JT;
    const int ch = blockIdx.y / JT;
    const int k0 = 1 + blockIdx.x * L::TX;
    const int j0 = jt * BY;
    const int i0 = i_begin + ch * chunk_len;
    const int i1 = min(i_end, i0 + chunk_len);
    if (i0 >= i1) {
        if (K2 == K_LAST && m.out_mode == WHB_OUT_FPI && tid == 0)
            m.partials[part_off + blockIdx.y * gridDim.x + blockIdx.x] = 0.0;
        return;
    }
    const long long S0 = g.S0;
    const int P = g.P;
    const int n_st = i1 - i0 + 4;  // staged planes i0-2 .. i1+1 (stage t <-> plane i0-2+t)

    if (tid == 0) {
        for (int q = 0; q < ST; ++q) {
            mbar_init(full + q, 1);
            mbar_init(empty + q, L::NA + L::NB);
        }
        for (int q = 0; q < 4; ++q) {
            mbar_init(e_full + q, L::NA);
            mbar_init(e_empty + q, L::NB);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int cl = 2 * lane;
    const int kx = k0 - 1 + cl;  // even global column of the lane pair
    const bool xin0 = kx >= 1 && kx < g.n2 - 1;
    const bool xin1 = kx + 1 >= 1 && kx + 1 < g.n2 - 1;
    double rsum = 0.0;

    if (warp == L::NA + L::NB) {
        // ---------------- producer
        if (lane == 0) {
            constexpr bool LOAD_P = (K1 != K_FIRST);
            constexpr uint32_t W_BYTES = (BY + 4) * L::WW * 8;
            constexpr uint32_t P_BYTES = L::ER * L::PW * 8;
            constexpr uint32_t A_BYTES = BY * L::PW * 8;
            constexpr uint32_t bytes = W_BYTES + (LOAD_P ? P_BYTES + A_BYTES : 0) + (ZF ? 0 : P_BYTES);
            for (int t = 0; t < n_st; ++t) {
                const int slot = t % ST;
                if (t >= ST) mbar_wait(empty + slot, ((t / ST) - 1) & 1);
                double *st = smem + (size_t)slot * L::STAGE;
                double *sp = st + L::W_EL, *sf = sp + L::P_EL, *sa = sf + L::P_EL;
                const int plane = i0 - 2 + t;
                mbar_expect_tx(full + slot, bytes);
                tma_load_3d(st, &tm_w, k0 - 3, j0 - 2, plane, full + slot);
                if (LOAD_P) {
                    tma_load_3d(sp, &tm_p, k0 - 1, j0 - 1, plane, full + slot);
                    tma_load_3d(sa, &tm_a, k0 - 1, j0, plane, full + slot);
                }
                if (!ZF) tma_load_3d(sf, &tm_f, k0 - 1, j0 - 1, plane, full + slot);
            }
        }
        __syncwarp();
    } else if (warp < L::NA) {
        // ---------------- group A: W^{s+1}(plane i), extended row ey = warp
        const double h1 = (K1 == K_FIRST) ? m.half_dt2 : m.dt2;
        const double cos1 = (K1 == K_FIRST) ? 1.0 : m.cos_f[s];
        const int ey = warp;
        const int jy = j0 - 1 + ey;
        const bool y1in = jy >= g.j_lo && jy < g.j_hi;
        const int rw = ey + 1, cw = cl + 2;
        for (int i = i0 - 1; i <= i1; ++i) {
            const int t = i - i0 + 2;
            const int e = i - (i0 - 1);  // E use index
            if (i == i0 - 1) {
                mbar_wait(full + ((t - 1) % ST), ((t - 1) / ST) & 1);
                mbar_wait(full + (t % ST), (t / ST) & 1);
            }
            mbar_wait(full + ((t + 1) % ST), ((t + 1) / ST) & 1);
            if (e >= 4) mbar_wait(e_empty + (e % 4), ((e / 4) - 1) & 1);
            const double *sm_m = smem + (size_t)((t - 1) % ST) * L::STAGE;
            const double *sm_c = smem + (size_t)(t % ST) * L::STAGE;
            const double *sm_p = smem + (size_t)((t + 1) % ST) * L::STAGE;
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
            if (K1 != K_FIRST) pv = *reinterpret_cast<const double2 *>(P_ + ey * L::PW + cl);
            const double a = update_point<K1, ZF, true>(g, wm.x, wc.x, wp.x, yl.x, yh.x, xl, wc.y, fv.x, pv.x, h1, cos1);
            const double b = update_point<K1, ZF, true>(g, wm.y, wc.y, wp.y, yl.y, yh.y, wc.x, xh, fv.y, pv.y, h1, cos1);
            const bool pin = (i >= g.i_lo) && (i < g.i_hi) && y1in;
            double *E = ering + (size_t)(e % 4) * L::E_EL;
            *reinterpret_cast<double2 *>(E + ey * L::WW + cw) = make_double2((pin && xin0) ? a : 0.0,
                                                                             (pin && xin1) ? b : 0.0);
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(e_full + (e % 4));
                mbar_arrive(empty + ((t - 1) % ST));  // last group-A use of plane i-1
            }
        }
        if (lane == 0) {  // planes i1 and i1+1 were never released by group A
            mbar_arrive(empty + ((i1 - i0 + 2) % ST));
            mbar_arrive(empty + ((i1 - i0 + 3) % ST));
        }
        __syncwarp();
    } else {
        // ---------------- group B: W^{s+2}(plane j), output row r = warp - NA
        const int r = warp - L::NA;
        const double cos2 = m.cos_f[s + 1];
        const double h2 = m.dt2;
        const double acc0 = m.acc_c[0], c1 = m.acc_c[s + 1], c2 = m.acc_c[s + 2];
        double *w1g = level_ptr(m, s + 1);
        double *w2g = level_ptr(m, s + 2);
        const int jo = j0 + r;
        const bool orow_ok = jo >= g.j_lo && jo < g.j_hi;
        const bool ok0 = orow_ok && xin0 && lane > 0;
        const bool ok1 = orow_ok && xin1 && lane < 31 && kx + 1 < k0 + L::TX;
        const int re = r + 1, cw = cl + 2;
        if (lane == 0) {  // group B never reads the stages of planes i0-2, i0-1: release them now (phase 0)
            mbar_arrive(empty + 0);
            mbar_arrive(empty + 1);
        }
        const bool want_v = (K2 == K_LAST) && m.out_mode != WHB_OUT_PLAIN && (ok0 || ok1);
        const long long pbase = (long long)jo * P + kx;
        double2 vcur = want_v ? *reinterpret_cast<const double2 *>(m.v + (long long)i0 * S0 + pbase)
                              : make_double2(0.0, 0.0);
        for (int j = i0; j < i1; ++j) {
            const double2 vnext = (want_v && j + 1 < i1)
                                      ? *reinterpret_cast<const double2 *>(m.v + (long long)(j + 1) * S0 + pbase)
                                      : make_double2(0.0, 0.0);
            const int e = j - (i0 - 1);  // E index of plane j
            const int t = j - i0 + 2;    // stage of plane j
            if (j == i0) {
                mbar_wait(e_full + ((e - 1) % 4), ((e - 1) / 4) & 1);
                mbar_wait(e_full + (e % 4), (e / 4) & 1);
            }
            mbar_wait(e_full + ((e + 1) % 4), ((e + 1) / 4) & 1);
            mbar_wait(full + (t % ST), (t / ST) & 1);
            const double *Em = ering + (size_t)((e - 1) % 4) * L::E_EL;
            const double *Ec = ering + (size_t)(e % 4) * L::E_EL;
            const double *Ep = ering + (size_t)((e + 1) % 4) * L::E_EL;
            const double *st_c = smem + (size_t)(t % ST) * L::STAGE;
            const double *F_ = st_c + L::W_EL + L::P_EL;
            const double *A_ = F_ + L::P_EL;
            const double2 e_c = *reinterpret_cast<const double2 *>(Ec + re * L::WW + cw);
            const double2 e_m = *reinterpret_cast<const double2 *>(Em + re * L::WW + cw);
            const double2 e_p = *reinterpret_cast<const double2 *>(Ep + re * L::WW + cw);
            const double2 e_yl = *reinterpret_cast<const double2 *>(Ec + (re - 1) * L::WW + cw);
            const double2 e_yh = *reinterpret_cast<const double2 *>(Ec + (re + 1) * L::WW + cw);
            const double e_xl = Ec[re * L::WW + cw - 1];
            const double e_xh = Ec[re * L::WW + cw + 2];
            const double2 w0 = *reinterpret_cast<const double2 *>(st_c + (r + 2) * L::WW + cw);
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
                const double2 ao = *reinterpret_cast<const double2 *>(A_ + r * L::PW + cl);
                a0 = whb_add(whb_add(ao.x, whb_mul(c1, e_c.x)), whb_mul(c2, n0));
                a1 = whb_add(whb_add(ao.y, whb_mul(c1, e_c.y)), whb_mul(c2, n1));
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(e_empty + ((e - 1) % 4));  // E plane j-1 is no longer needed
                mbar_arrive(empty + (t % ST));         // nor is the stage of plane j
            }
            const long long p = (long long)j * S0 + (long long)jo * P + kx;
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
            vcur = vnext;
        }
        if (lane == 0) {  // nor those of planes i1 and i1+1 (the producer has issued everything by now)
            mbar_arrive(empty + ((n_st - 2) % ST));
            mbar_arrive(empty + ((n_st - 1) % ST));
        }
        __syncwarp();
    }
    if (K2 == K_LAST && m.out_mode == WHB_OUT_FPI) {
        const double tsum = block_sum(rsum);
        if (tid == 0) m.partials[part_off + blockIdx.y * gridDim.x + blockIdx.x] = tsum;
    }
}

}  // namespace tb2w
