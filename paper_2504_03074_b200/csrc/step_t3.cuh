// Three leapfrog steps per HBM pass over a 3D grid (temporal blocking T = 3), TMA-pipelined,
// skewed so that ONE block barrier per plane orders everything (sm_100a).
//
// A CTA owns a BY x TX output tile (axis 1 x axis 2) and marches it through a chunk of axis-0
// planes [i0, i1).  Its 16 warps cover the level-1 region: warp w <-> row j0 - 2 + w, lane l <->
// the column pair k0 - 2 + 2l, +1 (64 columns).  Levels (time level s+t = "level t"):
//
//     level 1 on rows j0-2 .. j0+BY+1, columns k0-2 .. k0+TX+1   (16 x 64, halo 2)
//     level 2 on rows j0-1 .. j0+BY,   columns k0-1 .. k0+TX     (14 x 62, halo 1)
//     level 3 on rows j0   .. j0+BY-1, columns k0   .. k0+TX-1   (12 x 60, the tile)
//
// Iteration i computes level 1 at plane i, level 2 at plane i-2 and level 3 at plane i-4.  Every
// input of an iteration was produced by an EARLIER iteration (level 2 at i-2 reads level 1 at
// planes i-3..i-1; level 3 at i-4 reads level 2 at i-5..i-3), so the three level updates of an
// iteration are independent (3-way ILP per thread) and one split barrier per plane (an mbarrier:
// arrive after the level-1/2 stores, wait at the top of the next iteration) publishes them.  Axis-0 neighbours and the pointwise terms (W^{s-1}, f, the previous level, the filter
// sum) come from per-thread register queues; the axis-1/axis-2 neighbours of the level being
// stepped come from shared memory (W^s: the TMA stage; levels 1 and 2: 3-plane rings), axis-2
// neighbours inside a warp by shuffles.
//
// HBM traffic per output point per pass: read W^s, W^{s-1}, f, acc; write W^{s+2}, W^{s+3}, acc:
// 56 B for 3 updates = 18.7 B/update (28 for two steps per pass, 48 for one).  Halo boxes are
// re-read by the neighbouring tiles, mostly from L2.  Redundant level-1/2 work on the halo:
// (16*64 + 14*64) / (2*12*60) - 1 = 33 % of those two levels (the level-3 tile carries none).
//
// Arithmetic and its order are exactly three consecutive reference steps (update_point, the
// filter sum in step order), so the iterates stay bitwise equal to the reference's.
//
// Measured alternative (round 2): every stencil operand re-read from shared-memory level rings
// (5- / 4-plane rings, no register queues, f / acc / v from global one plane ahead) -- 164.5 vs
// 202.6 Gpts/s on config 4: the queue moves it saves cost less than the LDS->DMUL latency it adds
// (short-scoreboard stalls 24 % of samples vs barrier 19 %).
#pragma once

#include <type_traits>

// 1: the three level updates of an iteration interleaved (default); 0: one level after the other
#ifndef WHB_T3_ILP
#define WHB_T3_ILP 1
#endif

namespace t3 {

__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

using bulk::fence_proxy_async;
using bulk::mbar_expect_tx;
using bulk::mbar_init;
using bulk::mbar_wait;
using bulk::tma_load_3d;
using bulk::update_point;

constexpr int TX = 60;                 // output columns per tile
constexpr int BY = 12;                 // output rows per tile
constexpr int NR = BY + 4;             // level-1 rows (16): NR / R warps of R rows each
constexpr int LW = 64;                 // level-1 row width (columns k0-2 .. k0+61)
constexpr int RW = 68;                 // staged W^s row: columns k0-4 .. k0+63
constexpr int WR = BY + 6;             // staged W^s rows: j0-3 .. j0+BY+2
constexpr int W_EL = (WR * RW + 15) / 16 * 16;   // 1232 (128-B aligned sub-buffers for TMA)
constexpr int P_EL = NR * LW;                    // 1024: W^{s-1} / f box (the level-1 region)
constexpr int STAGE = W_EL + 2 * P_EL;           // 3280 doubles = 26.2 KB
constexpr int L1_EL = NR * LW;                   // level-1 plane
constexpr int L2_EL = (NR - 2) * LW;             // level-2 plane (rows j0-1 .. j0+BY)
constexpr int N2 = 4;                            // level-2 ring: planes i-5 .. i-2 (see the split barrier)

__device__ __forceinline__ void arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bulk::smem_u32(bar)) : "memory");
}

template <int ST>
constexpr size_t smem_bytes() {
    return (size_t)(ST * STAGE + 3 * L1_EL + N2 * L2_EL) * sizeof(double) + (ST + 1) * sizeof(uint64_t);
}

// Per-pass scalars (the reference's host expressions), passed as a kernel parameter.
struct Scal {
    double h1, cos1;            // step s (K_FIRST: dt^2/2 and 1)
    double cos2, cos3, dt2;     // steps s+1, s+2
    double c0, c1, c2, c3;      // filter weights acc_c[0], acc_c[s+1..s+3]
    double osc;                 // (2/T) dt (last pass)
};

// K1: kind of step s (FIRST when s == 0); K2: MID, or LAST when step s+2 ends the solve.
// GM: geometry mode as in tb2 / wf2d (0 generic, 1 equal taps, 2 equal taps and c^2 == 1).
template <int R>
constexpr int threads() {
    return 32 * NR / R;
}

// K1: kind of step s (FIRST when s == 0); K2: MID, or LAST when step s+2 ends the solve.
// GM: geometry mode as in tb2 / wf2d (0 generic, 1 equal taps, 2 equal taps and c^2 == 1).
// R: level-1 rows per warp (each lane: R rows x 2 columns); the axis-1 neighbours between a
// thread's own rows come from its registers, only the outer two from shared memory.
template <int ST, int K1, int K2, bool ZF, int GM, int R>
__global__ void __launch_bounds__(threads<R>(), 1)
    t3_kernel(Geom g, const Member *__restrict__ members, int s, int i_begin, int i_end, int chunk_len, int JT,
              const Scal sc, const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_p,
              const __grid_constant__ CUtensorMap tm_f) {
    constexpr bool SQ = GM >= 1;
    constexpr int C2M = GM == 2 ? 0 : -1;
    constexpr bool LOAD_P = (K1 != K_FIRST);
    static_assert(NR % R == 0, "rows per warp must divide the level-1 rows");
    extern __shared__ __align__(128) double smem[];
    double *l1buf = smem + (size_t)ST * STAGE;
    double *l2buf = l1buf + 3 * L1_EL;
    uint64_t *bars = reinterpret_cast<uint64_t *>(l2buf + N2 * L2_EL);
    uint64_t *itbar = bars + ST;  // per-plane split barrier: every thread arrives after its level 1/2 stores

    const Member m = members[0];
    const int w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // warp-uniform
    const int lane = threadIdx.x & 31;
    const int jt = blockIdx.y % JT;
    const int ch = blockIdx.y / JT;
    const int k0 = blockIdx.x * TX;
    const int j0 = jt * BY;
    const int i0 = i_begin + ch * chunk_len;
    const int i1 = min(i_end, i0 + chunk_len);
    if (i0 >= i1) {
        if (K2 == K_LAST && m.out_mode == WHB_OUT_FPI && threadIdx.x == 0)
            m.partials[blockIdx.y * gridDim.x + blockIdx.x] = 0.0;
        return;
    }
    double *w2g = level_ptr(m, s + 2);
    double *w3g = level_ptr(m, s + 3);
    const long long S0 = g.S0;
    const int P = g.P;

    constexpr uint32_t stage_bytes = (uint32_t)((RW * WR + (LOAD_P ? P_EL : 0) + (ZF ? 0 : P_EL)) * 8);
    // staged planes i0-3 .. i1+2; stage slot of plane p: (p - (i0 - 3)) % ST
    const int pfirst = i0 - 3;
    const int plast = i1 + 2;
    auto issue = [&](int plane) {
        const int slot = (plane - pfirst) % ST;
        double *st = smem + (size_t)slot * STAGE;
        uint64_t *bar = bars + slot;
        mbar_expect_tx(bar, stage_bytes);
        tma_load_3d(st, &tm_w, k0 - 4, j0 - 3, plane, bar);
        if (LOAD_P) tma_load_3d(st + W_EL, &tm_p, k0 - 2, j0 - 2, plane, bar);
        if (!ZF) tma_load_3d(st + W_EL + P_EL, &tm_f, k0 - 2, j0 - 2, plane, bar);
    };

    if (threadIdx.x == 0) {
        for (int t = 0; t < ST; ++t) mbar_init(bars + t, 1);
        mbar_init(itbar, 32 * NR / R);  // every thread of the CTA
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int p = pfirst; p <= plast && p < pfirst + ST; ++p) issue(p);
    }
    __syncthreads();

    // this thread's rows rho = w*R + r (level-1 region rows; y = j0 - 2 + rho) and column pair
    const int x = k0 - 2 + 2 * lane;
    const bool xin0 = (x >= 1) && (x < g.n2 - 1);
    const bool xin1 = (x + 1 >= 1) && (x + 1 < g.n2 - 1);
    const int rho0 = w * R;
    bool yin[R], ok0[R], ok1[R], yx0[R], yx1[R];
    long long pbase[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int y = j0 - 2 + rho0 + r;
        yin[r] = (y >= g.j_lo) && (y < g.j_hi);
        const bool own = (rho0 + r >= 2) && (rho0 + r <= NR - 3) && lane >= 1 && lane <= 30;
        ok0[r] = own && yin[r] && xin0;
        ok1[r] = own && yin[r] && xin1;
        yx0[r] = yin[r] && xin0;  // level value kept (not a Dirichlet / out-of-domain point)
        yx1[r] = yin[r] && xin1;
        pbase[r] = (long long)y * P + x;
    }
    bool any_ok = false;
#pragma unroll
    for (int r = 0; r < R; ++r) any_ok = any_ok || ok0[r] || ok1[r];
    // warp-uniform row ranges: level 2 on rows 1 .. NR-2, level 3 on rows 2 .. NR-3
    auto row2 = [&](int r) { return rho0 + r >= 1 && rho0 + r <= NR - 2; };
    auto row3 = [&](int r) { return rho0 + r >= 2 && rho0 + r <= NR - 3; };
    bool any2 = false, any3 = false;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        any2 = any2 || row2(r);
        any3 = any3 || row3(r);
    }
    const int wrow0 = (rho0 + 1) * RW + 2 + 2 * lane;  // first own row in a W^s stage
    const int prow0 = rho0 * LW + 2 * lane;            // first own row in a W^{s-1} / f box, level-1 plane

    auto plane_in = [&](int p) { return p >= g.i_lo && p < g.i_hi; };
    auto shl = [&](double v) { return __shfl_up_sync(0xffffffffu, v, 1); };
    auto shr = [&](double v) { return __shfl_down_sync(0xffffffffu, v, 1); };
    // Dirichlet / out-of-domain points of a level are 0 (one select per value)
    auto mask = [&](bool pin, double a, double b) -> double2 {
        return make_double2((pin && xin0) ? a : 0.0, (pin && xin1) ? b : 0.0);
    };
    auto lds2 = [&](const double *p) { return *reinterpret_cast<const double2 *>(p); };

    // register queues per own row (column pair): W^s at planes i+1 .. i-4, level 1 at i .. i-4,
    // level 2 at i-2 .. i-5, f at i .. i-4.  The plane loop is unrolled by ST = 6 (a multiple of
    // the level-ring period 3), so the queue shifts are register renames and every stage / ring
    // slot below is a compile-time constant.
    const double2 z2 = make_double2(0.0, 0.0);
    double2 ws0[R], ws1[R], ws2[R], ws3[R], ws4[R], ws5[R];  // ws0 = W^s(i+1), ws1 = W^s(i), ...
    double2 q10[R], q11[R], q12[R], q13[R], q14[R];          // q1k = level 1 at plane i-k
    double2 q20[R], q21[R], q22[R], q23[R];                  // q2k = level 2 at plane i-2-k
    double2 fq0[R], fq1[R], fq2[R], fq3[R], fq4[R];          // fqk = f at plane i-k
    double2 acc_n[R], v_n[R];
    double rsum = 0.0;

    // W^s centres of planes i0-3 and i0-2 (the first iteration, i = i0-2, adds plane i0-1); the
    // filter-sum input and v of the first output plane
    mbar_wait(bars + 0, 0);
    mbar_wait(bars + 1, 0);
    const bool want_v = (K2 == K_LAST) && m.out_mode != WHB_OUT_PLAIN;
    auto ld2 = [&](const double *base, int p, int r) -> double2 {
        return *reinterpret_cast<const double2 *>(base + (long long)p * S0 + pbase[r]);
    };
#pragma unroll
    for (int r = 0; r < R; ++r) {
        ws1[r] = lds2(smem + 0 * STAGE + wrow0 + r * RW);  // becomes W^s(i-1) below
        ws0[r] = lds2(smem + 1 * STAGE + wrow0 + r * RW);
        ws2[r] = ws3[r] = ws4[r] = ws5[r] = z2;
        q10[r] = q11[r] = q12[r] = q13[r] = q14[r] = z2;
        q20[r] = q21[r] = q22[r] = q23[r] = z2;
        fq0[r] = fq1[r] = fq2[r] = fq3[r] = fq4[r] = z2;
        acc_n[r] = (K1 != K_FIRST && (ok0[r] || ok1[r])) ? ld2(m.acc, i0, r) : z2;
        v_n[r] = (want_v && (ok0[r] || ok1[r])) ? ld2(m.v, i0, r) : z2;
        if (ok0[r] || ok1[r])
            for (int q = 1; q < 4 && i0 + q < i1; ++q) {
                if (K1 != K_FIRST) prefetch_l2(m.acc + (long long)(i0 + q) * S0 + pbase[r]);
                if (want_v) prefetch_l2(m.v + (long long)(i0 + q) * S0 + pbase[r]);
            }
    }
    __syncthreads();  // every thread has read plane pfirst: its slot takes plane pfirst + ST
    if (threadIdx.x == 0 && pfirst + ST <= plast) {
        fence_proxy_async();
        issue(pfirst + ST);
    }

    const int ibeg = i0 - 2;  // iteration i: level 1 at i, level 2 at i-2, level 3 at i-4
    const int iend = i1 + 3;
#if WHB_T3_ILP
    // Plane loop with the three level updates interleaved: every shared-memory operand of the
    // iteration (all written by earlier iterations) is loaded first, then the 3 x 2 x R update
    // chains are formed in one block (no memory operation between them, so the compiler
    // interleaves them: 6 independent fp64 chains per thread at R = 1 instead of 2), then levels 1
    // and 2 are published and the split barrier is arrived on, then the level-3 outputs.  The loop
    // is instantiated per warp role (warp-uniform): level 1 only (the outer two level-1 rows), levels
    // 1-2 (the next two), all three levels.
    auto run = [&](auto d2c, auto d3c) {
        constexpr bool D2 = decltype(d2c)::value;
        constexpr bool D3 = decltype(d3c)::value;
        int sl_i = 1 % ST, sl_n = 2 % ST, ph_n = 0;
        int r1w = 0, r12 = 1;
        int w2 = N2 - 2;
        for (int i = ibeg; i <= iend; ++i) {
            if (i > ibeg) {
                mbar_wait(itbar, (i - ibeg - 1) & 1);
                if (threadIdx.x == 0 && i - 1 + ST <= plast) {
                    fence_proxy_async();
                    issue(i - 1 + ST);
                }
            }
            const int SL_I = sl_i, SL_N = sl_n, R1W = r1w, R12 = r12, W2 = w2, R24 = (w2 + 2) % N2;
            if (i + 1 <= plast) mbar_wait(bars + SL_N, ph_n);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                ws5[r] = ws4[r]; ws4[r] = ws3[r]; ws3[r] = ws2[r]; ws2[r] = ws1[r]; ws1[r] = ws0[r];
                ws0[r] = lds2(smem + SL_N * STAGE + wrow0 + r * RW);
                q14[r] = q13[r]; q13[r] = q12[r]; q12[r] = q11[r]; q11[r] = q10[r];
                q23[r] = q22[r]; q22[r] = q21[r]; q21[r] = q20[r];
                fq4[r] = fq3[r]; fq3[r] = fq2[r]; fq2[r] = fq1[r]; fq1[r] = fq0[r];
            }
            // ---- operands: level 1 (W^s stage of plane i), level 2 (level-1 ring, plane i-2),
            //      level 3 (level-2 ring, plane i-4); x neighbours of levels 2 / 3 by shuffles
            const double *st = smem + SL_I * STAGE;
            const double2 y1lo = lds2(st + wrow0 - RW);
            const double2 y1hi = lds2(st + wrow0 + R * RW);
            double x1l[R], x1h[R];
            double2 pv[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int wrow = wrow0 + r * RW;
                x1l[r] = st[wrow - 1];
                x1h[r] = st[wrow + 2];
                const int prow = prow0 + r * LW;
                pv[r] = LOAD_P ? lds2(st + W_EL + prow) : z2;
                if (!ZF) fq0[r] = lds2(st + W_EL + P_EL + prow);
            }
            double2 y2lo = z2, y2hi = z2, y3lo = z2, y3hi = z2;
            double x2l[R], x2h[R], x3l[R], x3h[R];
            if (D2) {
                const double *l1 = l1buf + R12 * L1_EL;
                y2lo = lds2(l1 + (row2(0) ? prow0 - LW : prow0));
                y2hi = lds2(l1 + (row2(R - 1) ? prow0 + R * LW : prow0));
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    x2l[r] = shl(q12[r].y);
                    x2h[r] = shr(q12[r].x);
                }
            }
            if (D3) {
                const double *l2 = l2buf + R24 * L2_EL;
                y3lo = lds2(l2 + (row3(0) ? prow0 - 2 * LW : 2 * lane));
                y3hi = lds2(l2 + (row3(R - 1) ? prow0 + (R - 1) * LW : 2 * lane));
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    x3l[r] = shl(q22[r].y);
                    x3h[r] = shr(q22[r].x);
                }
            }
            // ---- the three level updates (independent chains)
            double a1[R], b1[R], a2[R], b2[R], a3[R], b3[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double2 yl = r == 0 ? y1lo : ws1[r - 1];
                const double2 yh = r == R - 1 ? y1hi : ws1[r + 1];
                a1[r] = update_point<K1, ZF, true, SQ, C2M>(g, ws2[r].x, ws1[r].x, ws0[r].x, yl.x, yh.x, x1l[r],
                                                         ws1[r].y, fq0[r].x, pv[r].x, sc.h1, sc.cos1);
                b1[r] = update_point<K1, ZF, true, SQ, C2M>(g, ws2[r].y, ws1[r].y, ws0[r].y, yl.y, yh.y, ws1[r].x,
                                                         x1h[r], fq0[r].y, pv[r].y, sc.h1, sc.cos1);
                if (D2) {
                    const double2 yl2 = r == 0 ? y2lo : q12[r - 1];
                    const double2 yh2 = r == R - 1 ? y2hi : q12[r + 1];
                    a2[r] = update_point<K_MID, ZF, true, SQ, C2M>(g, q13[r].x, q12[r].x, q11[r].x, yl2.x, yh2.x,
                                                                x2l[r], q12[r].y, fq2[r].x, ws3[r].x, sc.dt2, sc.cos2);
                    b2[r] = update_point<K_MID, ZF, true, SQ, C2M>(g, q13[r].y, q12[r].y, q11[r].y, yl2.y, yh2.y,
                                                                q12[r].x, x2h[r], fq2[r].y, ws3[r].y, sc.dt2, sc.cos2);
                }
                if (D3) {
                    const double2 yl3 = r == 0 ? y3lo : q22[r - 1];
                    const double2 yh3 = r == R - 1 ? y3hi : q22[r + 1];
                    a3[r] = update_point<K_MID, ZF, true, SQ, C2M>(g, q23[r].x, q22[r].x, q21[r].x, yl3.x, yh3.x,
                                                                x3l[r], q22[r].y, fq4[r].x, q14[r].x, sc.dt2, sc.cos3);
                    b3[r] = update_point<K_MID, ZF, true, SQ, C2M>(g, q23[r].y, q22[r].y, q21[r].y, yl3.y, yh3.y,
                                                                q22[r].x, x3h[r], fq4[r].y, q14[r].y, sc.dt2, sc.cos3);
                }
            }
            // ---- publish level 1 (plane i) and level 2 (plane i-2), then arrive
            const bool pin1 = plane_in(i);
            const bool pin2 = plane_in(i - 2);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int prow = prow0 + r * LW;
                const bool c0 = pin1 & yx0[r], c1 = pin1 & yx1[r];
                q10[r] = make_double2(c0 ? a1[r] : 0.0, c1 ? b1[r] : 0.0);
                *reinterpret_cast<double2 *>(l1buf + R1W * L1_EL + prow) = q10[r];
                if (D2 && row2(r)) {
                    const bool e0 = pin2 & yx0[r], e1 = pin2 & yx1[r];
                    q20[r] = make_double2(e0 ? a2[r] : 0.0, e1 ? b2[r] : 0.0);
                    *reinterpret_cast<double2 *>(l2buf + W2 * L2_EL + prow - LW) = q20[r];
                } else {
                    q20[r] = z2;
                }
            }
            arrive(itbar);

            // ---- level-3 outputs at plane i-4: the filter sum, W^{s+2}, W^{s+3}, acc (or v / dst)
            const int p3 = i - 4;
            const bool out3 = p3 >= i0 && p3 < i1;
            if (D3) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (!row3(r)) continue;
                    if (out3 && (ok0[r] || ok1[r])) {
                        // HBM -> L2 four planes ahead, so the one-plane-ahead register loads hit L2
                        if (p3 + 4 < i1) {
                            if (K1 != K_FIRST) prefetch_l2(m.acc + (long long)(p3 + 4) * S0 + pbase[r]);
                            if (want_v) prefetch_l2(m.v + (long long)(p3 + 4) * S0 + pbase[r]);
                        }
                        const double2 acc_c = acc_n[r], v_c = v_n[r];
                        double s0, s1;
                        if (K1 == K_FIRST) {  // timestep.py:284 then :298 per step
                            s0 = whb_add(whb_mul(sc.c0, ws5[r].x), whb_mul(sc.c1, q14[r].x));
                            s1 = whb_add(whb_mul(sc.c0, ws5[r].y), whb_mul(sc.c1, q14[r].y));
                        } else {
                            s0 = whb_add(acc_c.x, whb_mul(sc.c1, q14[r].x));
                            s1 = whb_add(acc_c.y, whb_mul(sc.c1, q14[r].y));
                        }
                        s0 = whb_add(whb_add(s0, whb_mul(sc.c2, q22[r].x)), whb_mul(sc.c3, a3[r]));
                        s1 = whb_add(whb_add(s1, whb_mul(sc.c2, q22[r].y)), whb_mul(sc.c3, b3[r]));
                        const long long p = (long long)p3 * S0 + pbase[r];
                        if (K2 == K_MID) {
                            if (ok0[r] && ok1[r]) {
                                *reinterpret_cast<double2 *>(w2g + p) = q22[r];
                                *reinterpret_cast<double2 *>(w3g + p) = make_double2(a3[r], b3[r]);
                                *reinterpret_cast<double2 *>(m.acc + p) = make_double2(s0, s1);
                            } else {
                                if (ok0[r]) { w2g[p] = q22[r].x; w3g[p] = a3[r]; m.acc[p] = s0; }
                                if (ok1[r]) { w2g[p + 1] = q22[r].y; w3g[p + 1] = b3[r]; m.acc[p + 1] = s1; }
                            }
                        } else {
                            const double o0 = whb_mul(sc.osc, s0);
                            const double o1 = whb_mul(sc.osc, s1);
                            if (m.out_mode == WHB_OUT_FPI) {
                                if (ok0[r]) { const double d = o0 - v_c.x; rsum += d * d; m.v[p] = o0; }
                                if (ok1[r]) { const double d = o1 - v_c.y; rsum += d * d; m.v[p + 1] = o1; }
                            } else if (m.out_mode == WHB_OUT_AV) {
                                if (ok0[r]) m.dst[p] = whb_sub(v_c.x, o0);
                                if (ok1[r]) m.dst[p + 1] = whb_sub(v_c.y, o1);
                            } else {
                                if (ok0[r]) m.dst[p] = o0;
                                if (ok1[r]) m.dst[p + 1] = o1;
                            }
                        }
                    }
                    // the next output plane's acc / v, after the last use of this plane's (so the
                    // load lands in the loop-carried registers), unconditionally and from an
                    // in-bounds plane (a predicated load merged with the old value made the compiler
                    // copy the loaded register right away, i.e. wait for the load)
                    const int pn = min(max(p3 + 1, i0), i1 - 1);
                    const long long o = (long long)pn * S0 + pbase[r];
                    if (K1 != K_FIRST) acc_n[r] = __ldcg(reinterpret_cast<const double2 *>(m.acc + o));
                    if (K2 == K_LAST) v_n[r] = __ldcg(reinterpret_cast<const double2 *>((want_v ? m.v : m.acc) + o));
                }
            }
            sl_i = sl_n;
            sl_n = sl_n + 1 == ST ? 0 : sl_n + 1;
            ph_n ^= (sl_n == 0);
            r1w = r12;
            r12 = (r12 + 1) % 3;
            w2 = w2 + 1 == N2 ? 0 : w2 + 1;
        }
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    if (any3) run(T_{}, T_{});
    else if (any2) run(T_{}, F_{});
    else run(F_{}, F_{});
#else
    // Plane loop, one copy of the body (a 6-way unrolled version with compile-time slots was
    // measured slower: 4-7K instructions of loop body thrash the instruction cache).  Stage and
    // ring slots advance incrementally: plane p <-> stage slot (p - pfirst) % ST.
    int sl_i = 1 % ST, sl_n = 2 % ST, ph_n = 0;  // stages of planes i and i+1, phase of the latter
    int r1w = 0, r12 = 1;  // level-1 ring (3 planes): slots of planes i and i-2
    int w2 = N2 - 2;       // level-2 ring (4 planes): slot of plane i-2 ((i - 2 - ibeg) mod 4)
    // Split per-plane barrier: a thread arrives on itbar right after its level-1 and level-2
    // stores of iteration i and waits for everybody's arrival only at the top of iteration i+1,
    // so the level-3 work of iteration i overlaps the barrier skew.  Safe because level 3 reads
    // only the level-2 ring, at plane i-4, and a thread can run at most the level-3 part ahead:
    // the level-2 store of iteration i+1 (plane i-1) lands in a different slot of the 4-plane ring;
    // the level-1 / stage slots rewritten at i+1 were last read before the arrivals of iteration i.
    for (int i = ibeg; i <= iend; ++i) {
        if (i > ibeg) {
            mbar_wait(itbar, (i - ibeg - 1) & 1);
            if (threadIdx.x == 0 && i - 1 + ST <= plast) {  // stage of plane i-1 is free
                fence_proxy_async();
                issue(i - 1 + ST);
            }
        }
        const int SL_I = sl_i, SL_N = sl_n, R1W = r1w, R12 = r12, W2 = w2, R24 = (w2 + 2) % N2;
        // shift the queues: plane i+1 of W^s enters
        // Every queue entry is assigned unconditionally in every copy (values outside a level's
        // plane range are computed from stale data and never stored or consumed), so the
        // compiler can rename the shifts instead of moving registers.
        if (i + 1 <= plast) mbar_wait(bars + SL_N, ph_n);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            ws5[r] = ws4[r]; ws4[r] = ws3[r]; ws3[r] = ws2[r]; ws2[r] = ws1[r]; ws1[r] = ws0[r];
            ws0[r] = lds2(smem + SL_N * STAGE + wrow0 + r * RW);
            q14[r] = q13[r]; q13[r] = q12[r]; q12[r] = q11[r]; q11[r] = q10[r];
            q23[r] = q22[r]; q22[r] = q21[r]; q21[r] = q20[r];
            fq4[r] = fq3[r]; fq3[r] = fq2[r]; fq2[r] = fq1[r]; fq1[r] = fq0[r];
        }

        // ---- level 1 at plane i (step s) on every row (needed for i <= i1 + 1)
        {
            const double *st = smem + SL_I * STAGE;
            const double2 ylo = lds2(st + wrow0 - RW);             // row rho0 - 1
            const double2 yhi = lds2(st + wrow0 + R * RW);         // row rho0 + R
            const bool pin = plane_in(i);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double2 yl = r == 0 ? ylo : ws1[r - 1];
                const double2 yh = r == R - 1 ? yhi : ws1[r + 1];
                const int wrow = wrow0 + r * RW;
                const double xl = st[wrow - 1], xh = st[wrow + 2];  // the stage has the halo columns
                const int prow = prow0 + r * LW;
                const double2 pv = LOAD_P ? lds2(st + W_EL + prow) : z2;
                if (!ZF) fq0[r] = lds2(st + W_EL + P_EL + prow);
                const double a = update_point<K1, ZF, true, SQ, C2M>(g, ws2[r].x, ws1[r].x, ws0[r].x, yl.x, yh.x, xl,
                                                                   ws1[r].y, fq0[r].x, pv.x, sc.h1, sc.cos1);
                const double b = update_point<K1, ZF, true, SQ, C2M>(g, ws2[r].y, ws1[r].y, ws0[r].y, yl.y, yh.y,
                                                                   ws1[r].x, xh, fq0[r].y, pv.y, sc.h1, sc.cos1);
                q10[r] = mask(pin && yin[r], a, b);
                *reinterpret_cast<double2 *>(l1buf + R1W * L1_EL + prow) = q10[r];
            }
        }

        // ---- level 2 at plane i-2 (step s+1): level 1 at i-3, i-2, i-1 (queues), rows rho-1, rho+1
        const int p2 = i - 2;  // needed for i0 - 1 <= p2 <= i1
        if (any2) {
            const double *l1 = l1buf + R12 * L1_EL;
            // (rows outside the level-2 region read in-bounds ring rows and are not used)
            const double2 ylo = lds2(l1 + (row2(0) ? prow0 - LW : prow0));
            const double2 yhi = lds2(l1 + (row2(R - 1) ? prow0 + R * LW : prow0));
            const bool pin = plane_in(p2);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (!row2(r)) {
                    q20[r] = z2;
                    continue;
                }
                const double2 yl = r == 0 ? ylo : q12[r - 1];
                const double2 yh = r == R - 1 ? yhi : q12[r + 1];
                const double xl = shl(q12[r].y), xh = shr(q12[r].x);
                // prev of step s+1 = W^s at plane i-2 (ws3), f at plane i-2 (fq2)
                const double a = update_point<K_MID, ZF, true, SQ, C2M>(g, q13[r].x, q12[r].x, q11[r].x, yl.x, yh.x,
                                                                      xl, q12[r].y, fq2[r].x, ws3[r].x, sc.dt2,
                                                                      sc.cos2);
                const double b = update_point<K_MID, ZF, true, SQ, C2M>(g, q13[r].y, q12[r].y, q11[r].y, yl.y, yh.y,
                                                                      q12[r].x, xh, fq2[r].y, ws3[r].y, sc.dt2,
                                                                      sc.cos2);
                q20[r] = mask(pin && yin[r], a, b);
                *reinterpret_cast<double2 *>(l2buf + W2 * L2_EL + prow0 + r * LW - LW) = q20[r];
            }
        }
        arrive(itbar);  // this thread's level-1 (plane i) and level-2 (plane i-2) stores are done

        // ---- level 3 at plane i-4 (step s+2) on the tile, then the filter sum and the outputs
        const int p3 = i - 4;
        const bool out3 = p3 >= i0 && p3 < i1;  // outputs (stores, residual, prefetch) only then
        if (any3) {
            const double *l2 = l2buf + R24 * L2_EL;
            const double2 ylo = lds2(l2 + (row3(0) ? prow0 - 2 * LW : 2 * lane));          // level-2 row rho0 - 1
            const double2 yhi = lds2(l2 + (row3(R - 1) ? prow0 + (R - 1) * LW : 2 * lane));  // row rho0 + R
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (!row3(r)) continue;
                const double2 yl = r == 0 ? ylo : q22[r - 1];
                const double2 yh = r == R - 1 ? yhi : q22[r + 1];
                const double xl = shl(q22[r].y), xh = shr(q22[r].x);
                // level 2 at i-5, i-4, i-3 = q23, q22, q21; prev = level 1 at i-4 (q14); f at i-4 (fq4)
                const double a3 = update_point<K_MID, ZF, true, SQ, C2M>(g, q23[r].x, q22[r].x, q21[r].x, yl.x, yh.x,
                                                                       xl, q22[r].y, fq4[r].x, q14[r].x, sc.dt2,
                                                                       sc.cos3);
                const double b3 = update_point<K_MID, ZF, true, SQ, C2M>(g, q23[r].y, q22[r].y, q21[r].y, yl.y, yh.y,
                                                                       q22[r].x, xh, fq4[r].y, q14[r].y, sc.dt2,
                                                                       sc.cos3);
                // next output plane's acc / v (one iteration ahead: hides the HBM latency)
                const double2 acc_c = acc_n[r], v_c = v_n[r];
                if (!out3 || !(ok0[r] || ok1[r])) continue;
                if (p3 + 1 < i1) {
                    if (K1 != K_FIRST) acc_n[r] = ld2(m.acc, p3 + 1, r);
                    if (want_v) v_n[r] = ld2(m.v, p3 + 1, r);
                }
                // HBM -> L2 four planes ahead, so the one-plane-ahead register loads above hit L2
                // (measured: without it 20 % of the warp samples waited on them)
                if (p3 + 4 < i1) {
                    if (K1 != K_FIRST) prefetch_l2(m.acc + (long long)(p3 + 4) * S0 + pbase[r]);
                    if (want_v) prefetch_l2(m.v + (long long)(p3 + 4) * S0 + pbase[r]);
                }
                // acc (+ c0 W^0 on the first pass) + c1 W^{s+1} + c2 W^{s+2} + c3 W^{s+3}, in step order
                double s0, s1;
                if (K1 == K_FIRST) {  // timestep.py:284 then :298 per step
                    s0 = whb_add(whb_mul(sc.c0, ws5[r].x), whb_mul(sc.c1, q14[r].x));
                    s1 = whb_add(whb_mul(sc.c0, ws5[r].y), whb_mul(sc.c1, q14[r].y));
                } else {
                    s0 = whb_add(acc_c.x, whb_mul(sc.c1, q14[r].x));
                    s1 = whb_add(acc_c.y, whb_mul(sc.c1, q14[r].y));
                }
                s0 = whb_add(whb_add(s0, whb_mul(sc.c2, q22[r].x)), whb_mul(sc.c3, a3));
                s1 = whb_add(whb_add(s1, whb_mul(sc.c2, q22[r].y)), whb_mul(sc.c3, b3));
                const long long p = (long long)p3 * S0 + pbase[r];
                if (K2 == K_MID) {
                    if (ok0[r] && ok1[r]) {
                        *reinterpret_cast<double2 *>(w2g + p) = q22[r];
                        *reinterpret_cast<double2 *>(w3g + p) = make_double2(a3, b3);
                        *reinterpret_cast<double2 *>(m.acc + p) = make_double2(s0, s1);
                    } else {
                        if (ok0[r]) { w2g[p] = q22[r].x; w3g[p] = a3; m.acc[p] = s0; }
                        if (ok1[r]) { w2g[p + 1] = q22[r].y; w3g[p + 1] = b3; m.acc[p + 1] = s1; }
                    }
                } else {
                    const double o0 = whb_mul(sc.osc, s0);
                    const double o1 = whb_mul(sc.osc, s1);
                    if (m.out_mode == WHB_OUT_FPI) {
                        if (ok0[r]) { const double d = o0 - v_c.x; rsum += d * d; m.v[p] = o0; }
                        if (ok1[r]) { const double d = o1 - v_c.y; rsum += d * d; m.v[p + 1] = o1; }
                    } else if (m.out_mode == WHB_OUT_AV) {
                        if (ok0[r]) m.dst[p] = whb_sub(v_c.x, o0);
                        if (ok1[r]) m.dst[p + 1] = whb_sub(v_c.y, o1);
                    } else {
                        if (ok0[r]) m.dst[p] = o0;
                        if (ok1[r]) m.dst[p + 1] = o1;
                    }
                }
            }
        }

        sl_i = sl_n;
        sl_n = sl_n + 1 == ST ? 0 : sl_n + 1;
        ph_n ^= (sl_n == 0);
        r1w = r12;  // (i+1) % 3 == (i-2) % 3
        r12 = (r12 + 1) % 3;
        w2 = w2 + 1 == N2 ? 0 : w2 + 1;
    }
#endif
    (void)any_ok;
    if (K2 == K_LAST && m.out_mode == WHB_OUT_FPI) {
        const double t = block_sum(rsum);
        if (threadIdx.x == 0) m.partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

}  // namespace t3
