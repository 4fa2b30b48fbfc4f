// Three leapfrog steps per HBM pass over a 3D grid (temporal blocking T = 3), TMA-pipelined,
// skewed so that ONE block barrier per plane orders everything (sm_100a).
//
// A CTA owns a BY x TX output tile (axis 1 x axis 2) and marches it through a chunk of axis-0
// planes [i0, i1).  Its 512 threads cover the level-1 region, one column pair per thread.  Tile
// shape (Shape<LX>, LX = lanes of a warp along axis 2; a warp covers 32 / LX rows):
//
//     LX = 32 (main): level-1 region 16 x 64, tile BY x TX = 12 x 60 (warp w <-> row j0 - 2 + w)
//     LX = 16 / 8 / 4 (ragged right edge): 32 x 32 / 64 x 16 / 128 x 8, tiles 28 x 28 / 60 x 12 / 124 x 4
//
// The last column of tiles of a grid whose interior width is not a multiple of 60 uses the
// narrowest shape that covers the remainder: on 1025^3 the remainder is 4 columns, which the main
// shape would serve with 86 x nch CTAs computing 64 columns each (5.5 % of the pass); the 124 x 4
// shape does it with 9 x nch.  Both shapes are bodies of the same kernel (one launch; the CTA
// picks by blockIdx.x), with the same arithmetic per point.  Levels (time level s+t = "level t"):
//
//     level 1 on rows j0-2 .. j0+BY+1, columns k0-2 .. k0+TX+1   (halo 2)
//     level 2 on rows j0-1 .. j0+BY,   columns k0-1 .. k0+TX     (halo 1)
//     level 3 on rows j0   .. j0+BY-1, columns k0   .. k0+TX-1   (the tile)
//
// Iteration i computes level 1 at plane i, level 2 at plane i-2 and level 3 at plane i-4.  Every
// input of an iteration was produced by an EARLIER iteration (level 2 at i-2 reads level 1 at
// planes i-3..i-1; level 3 at i-4 reads level 2 at i-5..i-3), so the three level updates of an
// iteration are independent (3-way ILP per thread) and one split barrier per plane (an mbarrier:
// arrive after the level-1/2 stores, wait at the top of the next iteration) publishes them.
// Axis-0 neighbours and the pointwise terms (W^{s-1}, f, the previous level, the filter sum) come
// from per-thread register queues; the axis-1 neighbours of the level being stepped come from
// shared memory (W^s: the TMA stage; levels 1 and 2: 3- / 4-plane rings), axis-2 neighbours of
// level 1 from the stage, of levels 2 / 3 by shuffles (a lane at the edge of its row receives a
// value of another row: it only feeds halo columns, which no output depends on).
//
// HBM traffic per output point per pass: read W^s, W^{s-1}, f, acc; write W^{s+2}, W^{s+3}, acc:
// 56 B for 3 updates = 18.7 B/update (28 for two steps per pass, 48 for one).  Halo boxes are
// re-read by the neighbouring tiles, mostly from L2.  Redundant level-1/2 work on the halo (main
// shape): (16*64 + 14*64) / (2*12*60) - 1 = 33 % of those two levels (the level-3 tile carries none).
//
// Arithmetic and its order are exactly three consecutive reference steps (update_point, the
// filter sum in step order), so the iterates stay bitwise equal to the reference's.
//
// Measured alternatives (round 2, config 4): every stencil operand re-read from shared-memory
// level rings (no register queues) 164.5 vs 202.6 Gpts/s; two rows per lane (8 warps) 120-160 vs
// 169-202; a 6-way unrolled plane loop 123-168 (instruction cache); the three level updates one
// after the other instead of interleaved 225.0 vs 236.7.
#pragma once

#include <type_traits>

// plane-loop unroll (measured on config 4: 1 -> 239.7, 2 -> 246.3, 3 -> 240.1 Gpts/s; 6 thrashes the instruction cache)
#ifndef WHB_T3_UNROLL
#define WHB_T3_UNROLL 2
#endif
#define T3_PRAGMA_(x) _Pragma(#x)
#define T3_UNROLL_(n) T3_PRAGMA_(unroll n)
#define T3_UNROLL(n) T3_UNROLL_(n)

// L2 policy experiments (config 4 is DRAM-bound at 6.0 TB/s on 77.6 GB per pass, 29 % above the
// compulsory bytes: the halo boxes of neighbouring tiles miss L2): WHB_T3_STCS streaming output
// stores, WHB_T3_LDCS streaming acc / v loads, WHB_T3_HINT evict-last TMA loads
#ifndef WHB_T3_STCS
#define WHB_T3_STCS 0
#endif
#ifndef WHB_T3_LDCS
#define WHB_T3_LDCS 0
#endif
#ifndef WHB_T3_HINT
#define WHB_T3_HINT 0
#endif
// L2 prefetch distance of the acc / v loads in planes (0: none)
#ifndef WHB_T3_PF
#define WHB_T3_PF 4
#endif

namespace t3 {

__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// tma_load_3d with an L2 cache-policy operand
__device__ __forceinline__ void tma_load_3d_hint(void *sdst, const CUtensorMap *map, int c0, int c1, int c2,
                                                 uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(bulk::smem_u32(sdst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bulk::smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void store2(double *p, double2 v) {
#if WHB_T3_STCS
    __stcs(reinterpret_cast<double2 *>(p), v);
#else
    *reinterpret_cast<double2 *>(p) = v;
#endif
}

__device__ __forceinline__ double2 load2_once(const double *p) {
#if WHB_T3_LDCS
    return __ldcs(reinterpret_cast<const double2 *>(p));
#else
    return __ldcg(reinterpret_cast<const double2 *>(p));
#endif
}

using bulk::fence_proxy_async;
using bulk::mbar_expect_tx;
using bulk::mbar_init;
using bulk::mbar_wait;
using bulk::tma_load_3d;
using bulk::update_point;

constexpr int NTHREADS = 512;          // 16 warps, one level-1 point pair per thread
constexpr int N2 = 4;                  // level-2 ring: planes i-5 .. i-2 (see the split barrier)

template <int LX>
struct Shape {
    static_assert(LX == 32 || LX == 16 || LX == 8 || LX == 4, "lanes along axis 2");
    static constexpr int RPW = 32 / LX;              // level-1 rows per warp
    static constexpr int NR = 16 * RPW;              // level-1 rows
    static constexpr int LW = 2 * LX;                // level-1 row width (columns k0-2 .. k0+TX+1)
    static constexpr int TX = LW - 4;                // output columns per tile
    static constexpr int BY = NR - 4;                // output rows per tile
    static constexpr int RW = LW + 4;                // staged W^s row: columns k0-4 .. k0+TX+3
    static constexpr int WR = NR + 2;                // staged W^s rows: j0-3 .. j0+BY+2
    static constexpr int W_EL = (WR * RW + 15) / 16 * 16;  // 128-B aligned sub-buffers for TMA
    static constexpr int P_EL = NR * LW;             // W^{s-1} / f box (the level-1 region): 1024
    static constexpr int A_EL = (BY * TX + 15) / 16 * 16;  // filter-sum box (the tile), of the plane 4 behind
    static constexpr int STAGE = W_EL + 2 * P_EL + A_EL;   // main: 4000 doubles = 32 KB
    static constexpr int L1_EL = NR * LW;            // level-1 plane
    static constexpr int L2_EL = (NR - 2) * LW;      // level-2 plane (rows j0-1 .. j0+BY)
    template <int ST>
    static constexpr size_t smem_bytes() {
        return (size_t)(ST * STAGE + 3 * L1_EL + N2 * L2_EL) * sizeof(double) + (ST + 1) * sizeof(uint64_t);
    }
};
using Main = Shape<32>;
constexpr int TX = Main::TX;           // main tile: 12 x 60
constexpr int BY = Main::BY;

// Shape of the last tile column for `rem` remaining interior columns (0: none left; 32: main).
constexpr int edge_lx(int rem) {
    return rem <= 0 ? 0 : rem <= Shape<4>::TX ? 4 : rem <= Shape<8>::TX ? 8 : rem <= Shape<16>::TX ? 16 : 32;
}

__device__ __forceinline__ void arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bulk::smem_u32(bar)) : "memory");
}

// Per-pass scalars (the reference's host expressions), passed as a kernel parameter.
struct Scal {
    double h1, cos1;            // step s (K_FIRST: dt^2/2 and 1)
    double cos2, cos3, dt2;     // steps s+1, s+2
    double c0, c1, c2, c3;      // filter weights acc_c[0], acc_c[s+1..s+3]
    double osc;                 // (2/T) dt (last pass)
};

// Row window of a launch: tile row jt starts at row j_off + jt * BY and only rows below j_end are
// written (whole grid: 0 and INT_MAX; the banded host iteration launches one band of rows per
// pass); part_off: first residual-partial slot of the launch.
struct RowWin {
    int j_off, j_end, part_off;
    int jt_fast;  // CTA -> tile order: row tiles fastest (1) or column tiles fastest (0, as launched)
};

// One CTA's march.  K1: kind of step s (FIRST when s == 0); K2: MID, or LAST when step s+2 ends
// the solve.  GM: geometry mode as in tb2 / wf2d (0 generic, 1 equal taps, 2 equal taps and
// c^2 == 1).  JT: row tiles of this shape; blockIdx.y = chunk * JTY + row tile (JTY = row tiles of
// the main shape, the grid's), k0: first output column.
template <int ST, int K1, int K2, bool ZF, int GM, int LX>
__device__ __forceinline__ void body(double *smem, const Geom &g, const Member *__restrict__ members, int s,
                                     int i_begin, int i_end, int chunk_len, int JTY, int JT, int yidx, int lin, int k0,
                                     const RowWin rw,
                                     const Scal &sc, const CUtensorMap *tm_w, const CUtensorMap *tm_p,
                                     const CUtensorMap *tm_f, const CUtensorMap *tm_a) {
    using S = Shape<LX>;
    constexpr int LW = S::LW, RW = S::RW, NR = S::NR, W_EL = S::W_EL, P_EL = S::P_EL, STAGE = S::STAGE;
    constexpr int L1_EL = S::L1_EL, L2_EL = S::L2_EL;
    constexpr bool UNI = (LX == 32);  // a warp is one row: the level roles are warp-uniform
    constexpr bool SQ = GM >= 1;
    constexpr int C2M = GM == 2 ? 0 : -1;
    constexpr bool LOAD_P = (K1 != K_FIRST);
    double *l1buf = smem + (size_t)ST * STAGE;
    double *l2buf = l1buf + 3 * L1_EL;
    uint64_t *bars = reinterpret_cast<uint64_t *>(l2buf + N2 * L2_EL);
    uint64_t *itbar = bars + ST;  // per-plane split barrier: every thread arrives after its level 1/2 stores

    const Member m = members[0];
    const int w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // warp-uniform
    const int lane = threadIdx.x & 31;
    const int cl = lane % LX;                  // column pair within the row
    const int rho = w * S::RPW + lane / LX;    // level-1 region row (y = j0 - 2 + rho)
    const int jt = yidx % JTY;  // yidx = chunk * JTY + row tile
    const int ch = yidx / JTY;
    const int j0 = rw.j_off + jt * S::BY;
    const int i0 = i_begin + ch * chunk_len;
    const int i1 = min(i_end, i0 + chunk_len);
    if (i0 >= i1 || jt >= JT) {
        if (K2 == K_LAST && m.out_mode == WHB_OUT_FPI && threadIdx.x == 0)
            m.partials[rw.part_off + lin] = 0.0;
        return;
    }
    double *w2g = level_ptr(m, s + 2);
    double *w3g = level_ptr(m, s + 3);
    const long long S0 = g.S0;
    const int P = g.P;

    constexpr int A_OFF = W_EL + 2 * P_EL;  // the filter sum of plane p - 4 rides in the stage of plane p
    constexpr uint32_t stage_bytes =
        (uint32_t)((RW * S::WR + (LOAD_P ? P_EL : 0) + (ZF ? 0 : P_EL) + (LOAD_P ? S::BY * S::TX : 0)) * 8);
    // staged planes i0-3 .. i1+2 (.. i1+3 when acc rides along: the last output plane's acc comes with
    // the stage of plane i1+3); stage slot of plane p: (p - (i0 - 3)) % ST
    const int pfirst = i0 - 3;
    const int plast = i1 + (LOAD_P ? 3 : 2);
#if WHB_T3_HINT
    const uint64_t pol = policy_evict_last();
#endif
    auto issue = [&](int plane) {
        const int slot = (plane - pfirst) % ST;
        double *st = smem + (size_t)slot * STAGE;
        uint64_t *bar = bars + slot;
        mbar_expect_tx(bar, stage_bytes);
#if WHB_T3_HINT
        tma_load_3d_hint(st, tm_w, k0 - 4, j0 - 3, plane, bar, pol);
        if (LOAD_P) tma_load_3d_hint(st + W_EL, tm_p, k0 - 2, j0 - 2, plane, bar, pol);
        if (!ZF) tma_load_3d_hint(st + W_EL + P_EL, tm_f, k0 - 2, j0 - 2, plane, bar, pol);
#else
        tma_load_3d(st, tm_w, k0 - 4, j0 - 3, plane, bar);
        if (LOAD_P) tma_load_3d(st + W_EL, tm_p, k0 - 2, j0 - 2, plane, bar);
        if (!ZF) tma_load_3d(st + W_EL + P_EL, tm_f, k0 - 2, j0 - 2, plane, bar);
#endif
        // acc of the plane whose outputs are formed while this stage is current (iteration `plane`)
        if (LOAD_P) tma_load_3d(st + A_OFF, tm_a, k0, j0, plane - 4, bar);
    };

    if (threadIdx.x == 0) {
        for (int t = 0; t < ST; ++t) mbar_init(bars + t, 1);
        mbar_init(itbar, NTHREADS);  // every thread of the CTA
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int p = pfirst; p <= plast && p < pfirst + ST; ++p) issue(p);
    }
    __syncthreads();

    // this thread's point pair
    const int x = k0 - 2 + 2 * cl;
    const int y = j0 - 2 + rho;
    const bool xin0 = (x >= 1) && (x < g.n2 - 1);
    const bool xin1 = (x + 1 >= 1) && (x + 1 < g.n2 - 1);
    const bool yin = (y >= g.j_lo) && (y < g.j_hi);
    const bool own = (rho >= 2) && (rho <= NR - 3) && cl >= 1 && cl <= LX - 2 && y < rw.j_end;
    const bool ok0 = own && yin && xin0;
    const bool ok1 = own && yin && xin1;
    const bool okk = ok0 || ok1;
    const bool yx0 = yin && xin0;  // level value kept (not a Dirichlet / out-of-domain point)
    const bool yx1 = yin && xin1;
    const long long pbase = (long long)y * P + x;
    // level 2 on region rows 1 .. NR-2, level 3 on rows 2 .. NR-3
    const bool r2 = rho >= 1 && rho <= NR - 2;
    const bool r3 = rho >= 2 && rho <= NR - 3;
    const int wlo = w * S::RPW, whi = wlo + S::RPW - 1;  // the warp's rows
    const bool any2 = whi >= 1 && wlo <= NR - 2;
    const bool any3 = whi >= 2 && wlo <= NR - 3;
    const int wrow0 = (rho + 1) * RW + 2 + 2 * cl;  // own row in a W^s stage
    const int prow0 = rho * LW + 2 * cl;            // own row in a W^{s-1} / f box, level-1 plane

    auto plane_in = [&](int p) { return p >= g.i_lo && p < g.i_hi; };
    auto shl = [&](double v) { return __shfl_up_sync(0xffffffffu, v, 1); };
    auto shr = [&](double v) { return __shfl_down_sync(0xffffffffu, v, 1); };
    auto lds2 = [&](const double *p) { return *reinterpret_cast<const double2 *>(p); };

    // register queues of the own column pair: W^s at planes i+1 .. i-4, level 1 at i .. i-4,
    // level 2 at i-2 .. i-5, f at i .. i-4
    const double2 z2 = make_double2(0.0, 0.0);
    double2 ws0, ws1, ws2, ws3, ws4, ws5;  // ws0 = W^s(i+1), ws1 = W^s(i), ...
    double2 q10, q11, q12, q13, q14;       // q1k = level 1 at plane i-k
    double2 q20, q21, q22, q23;            // q2k = level 2 at plane i-2-k
    double2 fq0, fq1, fq2, fq3, fq4;       // fqk = f at plane i-k
    double2 v_n;
    double rsum = 0.0;

    // W^s centres of planes i0-3 and i0-2 (the first iteration, i = i0-2, adds plane i0-1); the
    // filter-sum input and v of the first output plane
    mbar_wait(bars + 0, 0);
    mbar_wait(bars + 1, 0);
    const bool want_v = (K2 == K_LAST) && m.out_mode != WHB_OUT_PLAIN;
    auto ld2 = [&](const double *base, int p) -> double2 {
        return *reinterpret_cast<const double2 *>(base + (long long)p * S0 + pbase);
    };
    ws1 = lds2(smem + 0 * STAGE + wrow0);  // becomes W^s(i-1) below
    ws0 = lds2(smem + 1 * STAGE + wrow0);
    ws2 = ws3 = ws4 = ws5 = z2;
    q10 = q11 = q12 = q13 = q14 = z2;
    q20 = q21 = q22 = q23 = z2;
    fq0 = fq1 = fq2 = fq3 = fq4 = z2;
    v_n = (want_v && okk) ? ld2(m.v, i0) : z2;
    if (okk && want_v)
        for (int q = 1; q < WHB_T3_PF && i0 + q < i1; ++q) prefetch_l2(m.v + (long long)(i0 + q) * S0 + pbase);
    const int arow = (rho - 2) * S::TX + 2 * (cl - 1);  // own pair in the staged acc box (own threads only)
    __syncthreads();  // every thread has read plane pfirst: its slot takes plane pfirst + ST
    if (threadIdx.x == 0 && pfirst + ST <= plast) {
        fence_proxy_async();
        issue(pfirst + ST);
    }

    const int ibeg = i0 - 2;  // iteration i: level 1 at i, level 2 at i-2, level 3 at i-4
    const int iend = i1 + 3;
    // Plane loop with the three level updates interleaved: every shared-memory operand of the
    // iteration (all written by earlier iterations) is loaded first, then the 3 x 2 update chains
    // are formed in one block (no memory operation between them, so the compiler interleaves
    // them: 6 independent fp64 chains per thread), then levels 1 and 2 are published and the
    // split barrier is arrived on, then the level-3 outputs.  Split barrier: a thread arrives
    // right after its level-1 and level-2 stores of iteration i and waits for everybody's arrival
    // only at the top of iteration i+1, so the level-3 work of iteration i overlaps the barrier
    // skew.  Safe because level 3 reads only the level-2 ring, at plane i-4, and a thread can run
    // at most the level-3 part ahead: the level-2 store of iteration i+1 (plane i-1) lands in a
    // different slot of the 4-plane ring; the level-1 / stage slots rewritten at i+1 were last
    // read before the arrivals of iteration i.  The loop is instantiated per warp role
    // (warp-uniform): level 1 only (a warp of only outer level-1 rows), levels 1-2, all three.
    auto run = [&](auto d2c, auto d3c) {
        constexpr bool D2 = decltype(d2c)::value;
        constexpr bool D3 = decltype(d3c)::value;
        int sl_i = 1 % ST, sl_n = 2 % ST, ph_n = 0;  // stages of planes i and i+1, phase of the latter
        int r1w = 0, r12 = 1;                        // level-1 ring (3 planes): slots of planes i and i-2
        int w2 = N2 - 2;                             // level-2 ring (4 planes): slot of plane i-2
        T3_UNROLL(WHB_T3_UNROLL)
        for (int i = ibeg; i <= iend; ++i) {
            if (i > ibeg) {
                mbar_wait(itbar, (i - ibeg - 1) & 1);
                if (threadIdx.x == 0 && i - 1 + ST <= plast) {  // stage of plane i-1 is free
                    fence_proxy_async();
                    issue(i - 1 + ST);
                }
            }
            const int SL_I = sl_i, SL_N = sl_n, R1W = r1w, R12 = r12, W2 = w2, R24 = (w2 + 2) % N2;
            if (i + 1 <= plast) mbar_wait(bars + SL_N, ph_n);
            // shift the queues (every entry is assigned unconditionally, so the shifts rename)
            ws5 = ws4; ws4 = ws3; ws3 = ws2; ws2 = ws1; ws1 = ws0;
            ws0 = lds2(smem + SL_N * STAGE + wrow0);
            q14 = q13; q13 = q12; q12 = q11; q11 = q10;
            q23 = q22; q22 = q21; q21 = q20;
            fq4 = fq3; fq3 = fq2; fq2 = fq1; fq1 = fq0;
            // ---- operands: level 1 (W^s stage of plane i), level 2 (level-1 ring, plane i-2),
            //      level 3 (level-2 ring, plane i-4); x neighbours of levels 2 / 3 by shuffles
            const double *st = smem + SL_I * STAGE;
            const double2 y1lo = lds2(st + wrow0 - RW);
            const double2 y1hi = lds2(st + wrow0 + RW);
            const double x1l = st[wrow0 - 1];
            const double x1h = st[wrow0 + 2];
            const double2 pv = LOAD_P ? lds2(st + W_EL + prow0) : z2;
            if (!ZF) fq0 = lds2(st + W_EL + P_EL + prow0);
            // (read before the arrive: the stage is refilled once every thread has arrived)
            const double2 acc_c = (LOAD_P && D3 && own) ? lds2(st + A_OFF + arow) : z2;
            double2 y2lo = z2, y2hi = z2, y3lo = z2, y3hi = z2;
            double x2l = 0.0, x2h = 0.0, x3l = 0.0, x3h = 0.0;
            if (D2) {
                // (rows outside the level-2 region read in-bounds ring rows and are not used)
                const double *l1 = l1buf + R12 * L1_EL;
                y2lo = lds2(l1 + ((UNI || r2) ? prow0 - LW : prow0));
                y2hi = lds2(l1 + ((UNI || r2) ? prow0 + LW : prow0));
                x2l = shl(q12.y);
                x2h = shr(q12.x);
            }
            if (D3) {
                const double *l2 = l2buf + R24 * L2_EL;
                y3lo = lds2(l2 + ((UNI || r3) ? prow0 - 2 * LW : 2 * cl));  // level-2 row rho - 1
                y3hi = lds2(l2 + ((UNI || r3) ? prow0 : 2 * cl));           // level-2 row rho + 1
                x3l = shl(q22.y);
                x3h = shr(q22.x);
            }
            // ---- the three level updates (independent chains)
            double a2 = 0.0, b2 = 0.0, a3 = 0.0, b3 = 0.0;
            const double a1 = update_point<K1, ZF, true, SQ, C2M>(g, ws2.x, ws1.x, ws0.x, y1lo.x, y1hi.x, x1l, ws1.y,
                                                                fq0.x, pv.x, sc.h1, sc.cos1);
            const double b1 = update_point<K1, ZF, true, SQ, C2M>(g, ws2.y, ws1.y, ws0.y, y1lo.y, y1hi.y, ws1.x, x1h,
                                                                fq0.y, pv.y, sc.h1, sc.cos1);
            if (D2) {  // prev of step s+1 = W^s at plane i-2 (ws3), f at plane i-2 (fq2)
                a2 = update_point<K_MID, ZF, true, SQ, C2M>(g, q13.x, q12.x, q11.x, y2lo.x, y2hi.x, x2l, q12.y, fq2.x,
                                                          ws3.x, sc.dt2, sc.cos2);
                b2 = update_point<K_MID, ZF, true, SQ, C2M>(g, q13.y, q12.y, q11.y, y2lo.y, y2hi.y, q12.x, x2h, fq2.y,
                                                          ws3.y, sc.dt2, sc.cos2);
            }
            if (D3) {  // level 2 at i-5, i-4, i-3 = q23, q22, q21; prev = level 1 at i-4 (q14); f at i-4 (fq4)
                a3 = update_point<K_MID, ZF, true, SQ, C2M>(g, q23.x, q22.x, q21.x, y3lo.x, y3hi.x, x3l, q22.y, fq4.x,
                                                          q14.x, sc.dt2, sc.cos3);
                b3 = update_point<K_MID, ZF, true, SQ, C2M>(g, q23.y, q22.y, q21.y, y3lo.y, y3hi.y, q22.x, x3h, fq4.y,
                                                          q14.y, sc.dt2, sc.cos3);
            }
            // ---- publish level 1 (plane i) and level 2 (plane i-2), then arrive
            const bool pin1 = plane_in(i);
            const bool pin2 = plane_in(i - 2);
            {
                const bool c0 = pin1 & yx0, c1 = pin1 & yx1;
                q10 = make_double2(c0 ? a1 : 0.0, c1 ? b1 : 0.0);
                *reinterpret_cast<double2 *>(l1buf + R1W * L1_EL + prow0) = q10;
                if (D2 && (UNI || r2)) {
                    const bool e0 = pin2 & yx0, e1 = pin2 & yx1;
                    q20 = make_double2(e0 ? a2 : 0.0, e1 ? b2 : 0.0);
                    *reinterpret_cast<double2 *>(l2buf + W2 * L2_EL + prow0 - LW) = q20;
                } else {
                    q20 = z2;
                }
            }
            arrive(itbar);

            // ---- level-3 outputs at plane i-4: the filter sum, W^{s+2}, W^{s+3}, acc (or v / dst)
            const int p3 = i - 4;
            const bool out3 = p3 >= i0 && p3 < i1;
            if (D3 && (UNI || r3)) {
                if (out3 && okk) {
                    // HBM -> L2 four planes ahead, so the one-plane-ahead register loads hit L2
                    // (measured: without it 20 % of the warp samples waited on them)
                    if (WHB_T3_PF > 0 && want_v && p3 + WHB_T3_PF < i1)
                        prefetch_l2(m.v + (long long)(p3 + WHB_T3_PF) * S0 + pbase);
                    const double2 v_c = v_n;
                    // acc (+ c0 W^0 on the first pass) + c1 W^{s+1} + c2 W^{s+2} + c3 W^{s+3}, in step order
                    double s0, s1;
                    if (K1 == K_FIRST) {  // timestep.py:284 then :298 per step
                        s0 = whb_add(whb_mul(sc.c0, ws5.x), whb_mul(sc.c1, q14.x));
                        s1 = whb_add(whb_mul(sc.c0, ws5.y), whb_mul(sc.c1, q14.y));
                    } else {
                        s0 = whb_add(acc_c.x, whb_mul(sc.c1, q14.x));
                        s1 = whb_add(acc_c.y, whb_mul(sc.c1, q14.y));
                    }
                    s0 = whb_add(whb_add(s0, whb_mul(sc.c2, q22.x)), whb_mul(sc.c3, a3));
                    s1 = whb_add(whb_add(s1, whb_mul(sc.c2, q22.y)), whb_mul(sc.c3, b3));
                    const long long p = (long long)p3 * S0 + pbase;
                    if (K2 == K_MID) {
                        if (ok0 && ok1) {
                            store2(w2g + p, q22);
                            store2(w3g + p, make_double2(a3, b3));
                            store2(m.acc + p, make_double2(s0, s1));
                        } else {
                            if (ok0) { w2g[p] = q22.x; w3g[p] = a3; m.acc[p] = s0; }
                            if (ok1) { w2g[p + 1] = q22.y; w3g[p + 1] = b3; m.acc[p + 1] = s1; }
                        }
                    } else {
                        const double o0 = whb_mul(sc.osc, s0);
                        const double o1 = whb_mul(sc.osc, s1);
                        if (m.out_mode == WHB_OUT_FPI) {
                            if (ok0) { const double d = o0 - v_c.x; rsum += d * d; m.v[p] = o0; }
                            if (ok1) { const double d = o1 - v_c.y; rsum += d * d; m.v[p + 1] = o1; }
                        } else if (m.out_mode == WHB_OUT_AV) {
                            if (ok0) m.dst[p] = whb_sub(v_c.x, o0);
                            if (ok1) m.dst[p + 1] = whb_sub(v_c.y, o1);
                        } else {
                            if (ok0) m.dst[p] = o0;
                            if (ok1) m.dst[p + 1] = o1;
                        }
                    }
                }
                // the next output plane's acc / v, after the last use of this plane's (so the
                // load lands in the loop-carried registers), unconditionally and from an
                // in-bounds plane (a predicated load merged with the old value made the compiler
                // copy the loaded register right away, i.e. wait for the load)
                if (K2 == K_LAST) {
                    const int pn = min(max(p3 + 1, i0), i1 - 1);
                    v_n = load2_once((want_v ? m.v : m.acc) + (long long)pn * S0 + pbase);
                }
            }
            sl_i = sl_n;
            sl_n = sl_n + 1 == ST ? 0 : sl_n + 1;
            ph_n ^= (sl_n == 0);
            r1w = r12;  // (i+1) % 3 == (i-2) % 3
            r12 = (r12 + 1) % 3;
            w2 = w2 + 1 == N2 ? 0 : w2 + 1;
        }
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    if (any3) run(T_{}, T_{});
    else if (any2) run(T_{}, F_{});
    else run(F_{}, F_{});
    if (K2 == K_LAST && m.out_mode == WHB_OUT_FPI) {
        const double t = block_sum(rsum);
        if (threadIdx.x == 0) m.partials[rw.part_off + lin] = t;
    }
}

// LXE: shape of the last column of tiles (blockIdx.x == gridDim.x - 1); 32 = the main shape everywhere.
// The edge column has its own chunk length: in a one-wave launch (banded host iteration) its spare
// CTAs take shorter chunks, so the narrow tiles (more box rows per plane) are never the last to end.
template <int ST, int LXE>
constexpr size_t smem_bytes() {
    return Main::smem_bytes<ST>() > Shape<LXE>::template smem_bytes<ST>() ? Main::smem_bytes<ST>()
                                                                           : Shape<LXE>::template smem_bytes<ST>();
}

template <int ST, int K1, int K2, bool ZF, int GM, int LXE>
__global__ void __launch_bounds__(NTHREADS, 1)
    t3_kernel(Geom g, const Member *__restrict__ members, int s, int i_begin, int i_end, int chunk_len, int JT,
              int JTE, int chunk_len_e, const RowWin rw, const Scal sc, const __grid_constant__ CUtensorMap tm_w,
              const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_f,
              const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap te_w,
              const __grid_constant__ CUtensorMap te_p, const __grid_constant__ CUtensorMap te_f,
              const __grid_constant__ CUtensorMap te_a) {
    extern __shared__ __align__(128) double smem[];
    // CTA -> tile: the hardware starts CTAs in linear order (blockIdx.x fastest).  Column tiles
    // fastest (as launched) keeps the CTAs that run at the same time on whole grid rows: 262 vs 240
    // Gpts/s on 1025^3 against row tiles fastest (same DRAM bytes: CTAs 12 rows apart in one 480-B
    // column camp on the same channels); when a chunk's tiles all fit in one wave (257^3: 110) row
    // tiles fastest is ahead, 237 vs 227.
    const int lin = blockIdx.y * gridDim.x + blockIdx.x;
    int bx = blockIdx.x, yidx = blockIdx.y;
    if (rw.jt_fast) {
        const int per = gridDim.x * JT;
        const int chl = lin / per, r = lin - chl * per;
        bx = r / JT;
        yidx = chl * JT + (r - bx * JT);
    }
    if (LXE != 32 && bx == (int)gridDim.x - 1)
        // the edge column's JT * chunks CTAs: JTE row tiles x chunks of chunk_len_e planes (the rest exit)
        body<ST, K1, K2, ZF, GM, LXE>(smem, g, members, s, i_begin, i_end, chunk_len_e, JTE, JTE, yidx, lin,
                                      bx * Main::TX, rw, sc, &te_w, &te_p, &te_f, &te_a);
    else
        body<ST, K1, K2, ZF, GM, 32>(smem, g, members, s, i_begin, i_end, chunk_len, JT, JT, yidx, lin,
                                     bx * Main::TX, rw, sc, &tm_w, &tm_p, &tm_f, &tm_a);
}

}  // namespace t3
