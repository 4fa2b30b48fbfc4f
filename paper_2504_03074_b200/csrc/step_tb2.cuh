// Two leapfrog steps per pass over HBM (temporal blocking), TMA pipelined, sm_100a.
//
// A CTA owns a BY x TX tile (axis 1 x axis 2; BY = 1 in 2D) and marches it
// through a chunk of axis-0 planes.  For plane i it first computes W^{s+1} on
// the tile extended by one cell in y and x ("ext" tile, kept in a 3-plane
// shared-memory ring), then W^{s+2} on the tile at plane i-1 from the ring.
// Inputs per plane are staged by TMA exactly as in the one-step kernel, but
// with a 2-cell halo for W^s and a 1-cell halo for W^{s-1} and f:
//
//     read  W^s, W^{s-1}, f, acc          write W^{s+1}, W^{s+2}, acc
//
// i.e. 7 fp64 values per point for two updates (28 B/update instead of 48),
// plus the halo re-reads (served mostly from L2 because the neighbouring
// tiles march through the same planes at the same time).  Redundant work:
// W^{s+1} on the ext ring ((BY+2)(TX+2)/(BY TX) - 1 = 16% in 3D, <1% in 2D).
//
// Time levels live in a 4-slot ring (level_ptr): the pass reads levels s and
// s-1 and writes s+1 and s+2, so no CTA ever overwrites data another CTA of
// the same pass still reads.  Arithmetic and its order are exactly those of
// two consecutive reference steps (bitwise parity).
#pragma once

namespace tb2 {

using bulk::bulk_g2s;
using bulk::fence_proxy_async;
using bulk::mbar_expect_tx;
using bulk::mbar_init;
using bulk::mbar_wait;
using bulk::tma_load_3d;
using bulk::update_point;

constexpr int pad16(int x) { return (x + 15) / 16 * 16; }

template <int TX, int BY, bool A1>
struct Lay {
    static constexpr int RW = TX + 4;               // every staged row: columns k0-2 .. k0+TX+1
    static constexpr int WR = A1 ? BY + 4 : 1;      // W^s rows: j0-2 .. j0+BY+1
    static constexpr int ER = A1 ? BY + 2 : 1;      // ext rows: j0-1 .. j0+BY (prev, f, W^{s+1})
    static constexpr int W_EL = pad16(WR * RW);
    static constexpr int P_EL = pad16(ER * RW);
    static constexpr int A_EL = BY * TX;
    static constexpr int STAGE = W_EL + 2 * P_EL + A_EL;  // W^s | W^{s-1} | f | acc
    static constexpr int E_EL = pad16(ER * RW);
    static constexpr int THREADS = TX * BY / 2;
    static constexpr int RING = A1 ? 2 * (TX + 2) + 2 * BY : 2;  // ext-ring points, one per thread
};

template <int TX, int BY, int ST, bool A1>
constexpr size_t tb2_smem_bytes() {
    using L = Lay<TX, BY, A1>;
    return (size_t)(ST * L::STAGE + 3 * L::E_EL) * sizeof(double) + ST * sizeof(uint64_t);
}

// GM: geometry mode as in wf2d (0 generic; 1 equal taps on every axis: one centre product per
// point; 2 equal taps and c^2 == 1: no c^2 product).
template <int TX, int BY, int ST, bool A1, int K1, int K2, bool ZF, bool TENSOR, int GM = 0>
__global__ void __launch_bounds__(Lay<TX, BY, A1>::THREADS)
    tb2_kernel(Geom g, const Member *__restrict__ members, int member_off, int s, int i_begin, int i_end,
               int chunk_len, int JT, int part_off, int j_off, int j_end,
               const __grid_constant__ CUtensorMap tm_w,
               const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_f,
               const __grid_constant__ CUtensorMap tm_a) {
    using L = Lay<TX, BY, A1>;
    constexpr bool SQ = GM >= 1;
    constexpr int C2M = GM == 2 ? 0 : -1;
    static_assert(ST >= 4, "3 live planes + 1 in flight");
    static_assert(L::THREADS >= L::RING, "ext ring needs one thread per item");
    extern __shared__ __align__(128) double smem[];
    double *ering = smem + (size_t)ST * L::STAGE;
    uint64_t *bars = reinterpret_cast<uint64_t *>(ering + 3 * L::E_EL);

    const Member m = members[member_off + blockIdx.z];
    const int tid = threadIdx.x;
    const int jt = blockIdx.y % JT;
    const int ch = blockIdx.y / JT;
    const int k0 = blockIdx.x * TX;
    const int j0 = A1 ? j_off + jt * BY : 0;  // (j_off, j_end): row window of the launch, see t3::RowWin
    const int i0 = i_begin + ch * chunk_len;
    const int i1 = min(i_end, i0 + chunk_len);
    if (i0 >= i1) {
        if (K2 == K_LAST && m.out_mode == WHB_OUT_FPI && tid == 0)
            m.partials[part_off + blockIdx.y * gridDim.x + blockIdx.x] = 0.0;
        return;
    }
    const double *wcur = level_ptr(m, s);
    const double *wprv = level_ptr(m, s - 1);
    double *w1g = level_ptr(m, s + 1);
    double *w2g = level_ptr(m, s + 2);
    // step s (K1) and step s+1 (K2) scalars, as the reference forms them
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
    constexpr uint32_t W_BYTES = (TENSOR ? (TX + 4) * (BY + 4) : L::RW) * 8;
    constexpr uint32_t P_BYTES = (TENSOR ? (TX + 4) * (BY + 2) : L::RW) * 8;
    constexpr uint32_t A_BYTES = (TENSOR ? TX * BY : TX) * 8;
    constexpr uint32_t stage_bytes = W_BYTES + (LOAD_P ? P_BYTES : 0) + (ZF ? 0 : P_BYTES) + (LOAD_A ? A_BYTES : 0);
    // staged planes i0-2 .. i1+1; stage t <-> plane i0-2+t
    const int n_st = i1 - i0 + 4;

    auto issue = [&](int t) {
        const int slot = t % ST;
        double *st = smem + (size_t)slot * L::STAGE;
        double *sp = st + L::W_EL, *sf = sp + L::P_EL, *sa = sf + L::P_EL;
        uint64_t *bar = bars + slot;
        const int plane = i0 - 2 + t;
        mbar_expect_tx(bar, stage_bytes);
        if constexpr (TENSOR) {
            tma_load_3d(st, &tm_w, k0 - 2, j0 - 2, plane, bar);
            if (LOAD_P) tma_load_3d(sp, &tm_p, k0 - 2, j0 - 1, plane, bar);
            if (!ZF) tma_load_3d(sf, &tm_f, k0 - 2, j0 - 1, plane, bar);
            if (LOAD_A) tma_load_3d(sa, &tm_a, k0, j0, plane, bar);
        } else {  // 2D: one row segment per array
            const long long off = (long long)plane * S0 + (k0 - 2);
            bulk_g2s(st, wcur + off, L::RW * 8, bar);
            if (LOAD_P) bulk_g2s(sp, wprv + off, L::RW * 8, bar);
            if (!ZF) bulk_g2s(sf, m.f + off, L::RW * 8, bar);
            if (LOAD_A) bulk_g2s(sa, m.acc + off + 2, TX * 8, bar);
        }
    };

    if (tid == 0) {
        for (int t = 0; t < ST; ++t) mbar_init(bars + t, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const int pro = min(n_st, ST);
        for (int t = 0; t < pro; ++t) issue(t);
    }
    __syncthreads();

    // main pair of this thread
    const int ty = A1 ? tid / (TX / 2) : 0;
    const int kl = 2 * (A1 ? tid % (TX / 2) : tid);
    const int j = j0 + ty;
    const int k = k0 + kl;
    const bool row_ok = !A1 || (j >= g.j_lo && j < g.j_hi);
    const bool ok0 = row_ok && (k >= 1) && (k < g.n2 - 1);
    const bool ok1 = row_ok && (k + 1 < g.n2 - 1);
    const bool st0 = ok0 && (j < j_end);  // stored (ok0 / ok1 also keep W^{s+1} on rows past the window)
    const bool st1 = ok1 && (j < j_end);
    // ext-ring item of this thread (3D: top/bottom row pairs, then left/right singles; 2D: 2 singles)
    int r_ey = 0, r_ex = 0;
    bool r_pair = false, r_any = false;
    if (A1) {
        // one ring point per thread for the first RING threads (the barrier after the W^{s+1}
        // phase waits for the slowest thread: 3 points, not 4 as with pairs on the top/bottom rows)
        if (tid < 2 * (TX + 2)) {
            r_any = true;
            r_ey = (tid < TX + 2) ? -1 : BY;
            r_ex = (tid % (TX + 2)) - 1;
        } else if (tid < L::RING) {
            r_any = true;
            const int q = tid - 2 * (TX + 2);
            r_ex = (q < BY) ? -1 : TX;
            r_ey = q % BY;
        }
    } else if (tid < 2) {
        r_any = true;
        r_ex = tid == 0 ? -1 : TX;
    }
    double rsum = 0.0;

    // W^{s+1} at ext point (ey, ex) of plane i from stages (tm, tc, tp)
    auto step1 = [&](const double *sm_m, const double *sm_c, const double *sm_p, int i, int ey, int ex) -> double {
        const int r = A1 ? ey + 2 : 0;
        const int c = ex + 2;
        const int re = A1 ? ey + 1 : 0;
        const double *P_ = sm_c + L::W_EL;
        const double *F_ = P_ + L::P_EL;
        const double wc = sm_c[r * L::RW + c];
        const double yl = A1 ? sm_c[(r - 1) * L::RW + c] : 0.0;
        const double yh = A1 ? sm_c[(r + 1) * L::RW + c] : 0.0;
        const double fv = ZF ? 0.0 : F_[re * L::RW + c];
        const double pv = LOAD_P ? P_[re * L::RW + c] : 0.0;
        const double w = update_point<K1, ZF, A1, SQ, C2M>(g, sm_m[r * L::RW + c], wc, sm_p[r * L::RW + c], yl, yh,
                                                 sm_c[r * L::RW + c - 1], sm_c[r * L::RW + c + 1], fv, pv, h1, cos1);
        const int jj = j0 + ey, kk = k0 + ex;
        const bool inside = (i >= g.i_lo) && (i < g.i_hi) && (kk >= 1) && (kk < g.n2 - 1) &&
                            (!A1 || (jj >= g.j_lo && jj < g.j_hi));
        return inside ? w : 0.0;  // Dirichlet (and out-of-domain) points of W^{s+1} are 0
    };

    // last pass: v of the next output plane is loaded one iteration ahead (hides its HBM latency)
    const bool want_v = (K2 == K_LAST) && m.out_mode != WHB_OUT_PLAIN && row_ok && (st0 || st1);
    const long long pbase = (long long)j * P + k;
    double2 vcur = make_double2(0.0, 0.0);
    // register queues along axis 0 for the main pair: W^s at planes i-1, i and W^{s+1} at
    // planes i-2, i-1 (each value was read from / written to shared memory by this thread)
    double2 wsm = make_double2(0.0, 0.0), wsc = wsm, em2 = wsm, em1 = wsm;
    const int rmain = (A1 ? ty + 2 : 0) * L::RW + kl + 2;  // main pair in a W^s stage
    const int emain = (A1 ? ty + 1 : 0) * L::RW + kl + 2;  // main pair in an E slot / prev / f row
    for (int i = i0 - 1; i <= i1; ++i) {
        const int t = i - i0 + 2;  // stage of plane i
        // output plane of this iteration is i-1; prefetch v for plane i (next iteration's output)
        const double2 vnext = (want_v && i >= i0 && i < i1)
                                  ? *reinterpret_cast<const double2 *>(m.v + (long long)i * S0 + pbase)
                                  : make_double2(0.0, 0.0);
        if (i > i0 - 1) {
            __syncthreads();  // plane i-1 done: stage of plane i-2 and E slot of plane i-3 are free
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

        // ---- step s: W^{s+1}(plane i) on the ext tile -> E ring
        double2 enew, wsp;
        {
            if (i == i0 - 1) {
                wsm = *reinterpret_cast<const double2 *>(sm_m + rmain);
                wsc = *reinterpret_cast<const double2 *>(sm_c + rmain);
            }
            wsp = *reinterpret_cast<const double2 *>(sm_p + rmain);
            const double *P_ = sm_c + L::W_EL;
            const double *F_ = P_ + L::P_EL;
            double2 yl2 = make_double2(0.0, 0.0), yh2 = yl2;
            if (A1) {
                yl2 = *reinterpret_cast<const double2 *>(sm_c + rmain - L::RW);
                yh2 = *reinterpret_cast<const double2 *>(sm_c + rmain + L::RW);
            }
            const double xl = sm_c[rmain - 1], xh = sm_c[rmain + 2];
            const double2 fv2 = ZF ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2 *>(F_ + emain);
            const double2 pv2 = LOAD_P ? *reinterpret_cast<const double2 *>(P_ + emain) : make_double2(0.0, 0.0);
            const double a = update_point<K1, ZF, A1, SQ, C2M>(g, wsm.x, wsc.x, wsp.x, yl2.x, yh2.x, xl, wsc.y, fv2.x, pv2.x,
                                                     h1, cos1);
            const double b = update_point<K1, ZF, A1, SQ, C2M>(g, wsm.y, wsc.y, wsp.y, yl2.y, yh2.y, wsc.x, xh, fv2.y, pv2.y,
                                                     h1, cos1);
            const bool pin = (i >= g.i_lo) && (i < g.i_hi);
            enew = make_double2((pin && ok0) ? a : 0.0, (pin && ok1) ? b : 0.0);
            *reinterpret_cast<double2 *>(E + emain) = enew;
        }
        if (r_any) {
            const double a = step1(sm_m, sm_c, sm_p, i, r_ey, r_ex);
            E[(A1 ? r_ey + 1 : 0) * L::RW + r_ex + 2] = a;
            if (r_pair) E[(A1 ? r_ey + 1 : 0) * L::RW + r_ex + 3] = step1(sm_m, sm_c, sm_p, i, r_ey, r_ex + 1);
        }
        __syncthreads();

        // ---- step s+1: W^{s+2}(plane i-1) on the tile
        const int ip = i - 1;
        if (ip >= i0) {
            const double *Ec = ering + (size_t)(ip % 3) * L::E_EL;
            const double *st_c = sm_m;                                     // stage of plane ip
            const double *F_ = st_c + L::W_EL + L::P_EL;
            const double *A_ = F_ + L::P_EL;
            const int re = A1 ? ty + 1 : 0;
            const int c = kl + 2;
            const double2 e_c = em1;  // W^{s+1} at planes ip, ip-1, ip+1 (register queue)
            const double2 e_m = em2;
            const double2 e_p = enew;
            double2 e_yl = make_double2(0.0, 0.0), e_yh = make_double2(0.0, 0.0);
            if (A1) {
                e_yl = *reinterpret_cast<const double2 *>(Ec + (re - 1) * L::RW + c);
                e_yh = *reinterpret_cast<const double2 *>(Ec + (re + 1) * L::RW + c);
            }
            const double e_xl = Ec[re * L::RW + c - 1];
            const double e_xh = Ec[re * L::RW + c + 2];
            const double2 w0 = wsm;  // W^s at plane ip (prev of step s+1)
            const double2 f2 = ZF ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2 *>(F_ + re * L::RW + c);
            const double n0 = update_point<K_MID, ZF, A1, SQ, C2M>(g, e_m.x, e_c.x, e_p.x, e_yl.x, e_yh.x, e_xl, e_c.y, f2.x,
                                                         w0.x, h2, cos2);
            const double n1 = update_point<K_MID, ZF, A1, SQ, C2M>(g, e_m.y, e_c.y, e_p.y, e_yl.y, e_yh.y, e_c.x, e_xh, f2.y,
                                                         w0.y, h2, cos2);
            double a0, a1;
            if (K1 == K_FIRST) {  // acc = c0*W^0 + c1*W^1, then += c2*W^2   (timestep.py:284, 298)
                a0 = whb_add(whb_add(whb_mul(acc0, w0.x), whb_mul(c1, e_c.x)), whb_mul(c2, n0));
                a1 = whb_add(whb_add(whb_mul(acc0, w0.y), whb_mul(c1, e_c.y)), whb_mul(c2, n1));
            } else {
                const double2 ao = *reinterpret_cast<const double2 *>(A_ + ty * TX + kl);
                a0 = whb_add(whb_add(ao.x, whb_mul(c1, e_c.x)), whb_mul(c2, n0));
                a1 = whb_add(whb_add(ao.y, whb_mul(c1, e_c.y)), whb_mul(c2, n1));
            }
            const long long p = (long long)ip * S0 + (long long)j * P + k;
            if (K2 == K_MID) {
                if (st0 && st1) {
                    *reinterpret_cast<double2 *>(w1g + p) = e_c;
                    *reinterpret_cast<double2 *>(w2g + p) = make_double2(n0, n1);
                    *reinterpret_cast<double2 *>(m.acc + p) = make_double2(a0, a1);
                } else {
                    if (st0) { w1g[p] = e_c.x; w2g[p] = n0; m.acc[p] = a0; }
                    if (st1) { w1g[p + 1] = e_c.y; w2g[p + 1] = n1; m.acc[p + 1] = a1; }
                }
            } else {
                const double o0 = whb_mul(m.out_scale, a0);
                const double o1 = whb_mul(m.out_scale, a1);
                if (m.out_mode == WHB_OUT_FPI) {
                    if (st0) {
                        const double d0 = o0 - vcur.x;
                        rsum += d0 * d0;
                        m.v[p] = o0;
                    }
                    if (st1) {
                        const double d1 = o1 - vcur.y;
                        rsum += d1 * d1;
                        m.v[p + 1] = o1;
                    }
                } else if (m.out_mode == WHB_OUT_AV) {
                    if (st0) m.dst[p] = whb_sub(vcur.x, o0);
                    if (st1) m.dst[p + 1] = whb_sub(vcur.y, o1);
                } else {
                    if (st0) m.dst[p] = o0;
                    if (st1) m.dst[p + 1] = o1;
                }
            }
        }
        vcur = vnext;
        wsm = wsc;
        wsc = wsp;
        em2 = em1;
        em1 = enew;
    }
    if (K2 == K_LAST && m.out_mode == WHB_OUT_FPI) {
        const double t = block_sum(rsum);
        if (tid == 0) m.partials[part_off + blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

}  // namespace tb2
