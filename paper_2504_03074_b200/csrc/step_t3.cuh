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
// iteration are independent (3-way ILP per thread) and one __syncthreads per plane publishes
// them.
//
// Every stencil operand is read from shared memory where it was stored once: W^s from the TMA
// stage ring (planes i-2 .. i+1 live, the next planes in flight), level 1 from a 5-plane ring
// (i-4 .. i), level 2 from a 4-plane ring (i-5 .. i-2) -- axis-0 neighbours and the thread's own
// centre value included, so nothing is carried across iterations in registers (measured: the
// register-queue version spent a fifth of its instructions on queue moves).  Axis-2 neighbours of
// levels 2 and 3 come from warp shuffles.  The pointwise streams -- f at planes i, i-2, i-4, the
// filter sum acc and v at the output plane -- are loaded straight from global memory one
// iteration ahead, with an L2 prefetch four planes ahead of that (f of the two later uses is an
// L2 hit: the first use brought it in).
//
// HBM traffic per output point per pass: read W^s, W^{s-1}, f, acc; write W^{s+2}, W^{s+3}, acc:
// 56 B for 3 updates = 18.7 B/update (28 for two steps per pass, 48 for one).  Halo boxes are
// re-read by the neighbouring tiles, mostly from L2.  Redundant level-1/2 work on the halo:
// (16*64 + 14*64) / (2*12*60) - 1 = 33 % of those two levels (the level-3 tile carries none).
//
// Arithmetic and its order are exactly three consecutive reference steps (update_point, the
// filter sum in step order), so the iterates stay bitwise equal to the reference's.
#pragma once

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
constexpr int NR = BY + 4;             // level-1 rows = warps (16)
constexpr int THREADS = 32 * NR;       // 512
constexpr int LW = 64;                 // level-1 row width (columns k0-2 .. k0+61)
constexpr int RW = 68;                 // staged W^s row: columns k0-4 .. k0+63
constexpr int WR = BY + 6;             // staged W^s rows: j0-3 .. j0+BY+2
constexpr int W_EL = (WR * RW + 15) / 16 * 16;   // 1232 (128-B aligned sub-buffers for TMA)
constexpr int P_EL = NR * LW;                    // 1024: W^{s-1} box (the level-1 region)
constexpr int STAGE = W_EL + P_EL;               // 2256 doubles = 18 KB
constexpr int L1_EL = NR * LW;                   // level-1 plane
constexpr int L2_EL = (NR - 2) * LW;             // level-2 plane (rows j0-1 .. j0+BY)
constexpr int N1 = 5;                            // level-1 ring: planes i-4 .. i
constexpr int N2 = 4;                            // level-2 ring: planes i-5 .. i-2

template <int ST>
constexpr size_t smem_bytes() {
    return (size_t)(ST * STAGE + N1 * L1_EL + N2 * L2_EL) * sizeof(double) + ST * sizeof(uint64_t);
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
template <int ST, int K1, int K2, bool ZF, int GM>
__global__ void __launch_bounds__(THREADS, 1)
    t3_kernel(Geom g, const Member *__restrict__ members, int s, int i_begin, int i_end, int chunk_len, int JT,
              const Scal sc, const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_p) {
    constexpr bool SQ = GM >= 1;
    constexpr int C2M = GM == 2 ? 0 : -1;
    constexpr bool LOAD_P = (K1 != K_FIRST);
    static_assert(ST >= 6, "W^s planes i-2 .. i+1 live and at least two in flight");
    extern __shared__ __align__(128) double smem[];
    double *l1buf = smem + (size_t)ST * STAGE;
    double *l2buf = l1buf + N1 * L1_EL;
    uint64_t *bars = reinterpret_cast<uint64_t *>(l2buf + N2 * L2_EL);

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
    const double *f = m.f;
    const long long S0 = g.S0;
    const int P = g.P;

    constexpr uint32_t stage_bytes = (uint32_t)((RW * WR + (LOAD_P ? P_EL : 0)) * 8);
    // staged planes i0-3 .. i1+2; stage slot of plane p: (p - (i0 - 3)) % ST.  A stage's last
    // reader is level 2, two iterations after the plane's own iteration.
    const int pfirst = i0 - 3;
    const int plast = i1 + 2;
    auto issue = [&](int plane) {
        const int slot = (plane - pfirst) % ST;
        double *st = smem + (size_t)slot * STAGE;
        uint64_t *bar = bars + slot;
        mbar_expect_tx(bar, stage_bytes);
        tma_load_3d(st, &tm_w, k0 - 4, j0 - 3, plane, bar);
        if (LOAD_P) tma_load_3d(st + W_EL, &tm_p, k0 - 2, j0 - 2, plane, bar);
    };

    if (threadIdx.x == 0) {
        for (int t = 0; t < ST; ++t) mbar_init(bars + t, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int p = pfirst; p <= plast && p < pfirst + ST; ++p) issue(p);
    }
    __syncthreads();

    // this thread's row / column pair
    const int y = j0 - 2 + w;
    const int x = k0 - 2 + 2 * lane;
    const bool yin = (y >= g.j_lo) && (y < g.j_hi);
    const bool xin0 = (x >= 1) && (x < g.n2 - 1);
    const bool xin1 = (x + 1 >= 1) && (x + 1 < g.n2 - 1);
    const bool do2 = (w >= 1) && (w <= NR - 2);        // warp-uniform: rows of level 2
    const bool do3 = (w >= 2) && (w <= NR - 3);        // rows of level 3 (the output tile)
    const bool own = do3 && lane >= 1 && lane <= 30;   // output points: the tile, interior only
    const bool ok0 = own && yin && xin0;
    const bool ok1 = own && yin && xin1;
    const bool okp = ok0 || ok1;
    const int wrow = (w + 1) * RW + 2 + 2 * lane;      // this pair in a W^s stage
    const int prow = w * LW + 2 * lane;                // this pair in a W^{s-1} box / level-1 plane
    const int qrow = prow - LW;                        // this pair in a level-2 plane
    const long long pbase = (long long)y * P + x;

    auto plane_in = [&](int p) { return p >= g.i_lo && p < g.i_hi; };
    auto shl = [&](double v) { return __shfl_up_sync(0xffffffffu, v, 1); };
    auto shr = [&](double v) { return __shfl_down_sync(0xffffffffu, v, 1); };
    auto lds2 = [&](const double *p) { return *reinterpret_cast<const double2 *>(p); };
    auto sts2 = [&](double *p, double2 v) { *reinterpret_cast<double2 *>(p) = v; };
    auto mask = [&](bool pin, double a, double b) -> double2 {
        return make_double2((pin && xin0) ? a : 0.0, (pin && xin1) ? b : 0.0);
    };
    const double2 z2 = make_double2(0.0, 0.0);
    const bool want_v = (K2 == K_LAST) && m.out_mode != WHB_OUT_PLAIN;
    const bool need_v = want_v || K1 == K_FIRST;  // W^0 = v enters the first pass's filter sum
    // pointwise global streams as running pointers (one plane = S0 elements), loaded one iteration
    // ahead under warp-uniform "needed" conditions, so every address is inside the allocation:
    // f at planes i (level 1, needed for i <= i1+1), i-2 (level 2, for i0-1 <= i-2 <= i1) and i-4
    // (level 3, for i0 <= i-4 < i1); acc and v at the output plane i-4.  f is read-only in the
    // kernel (non-coherent path); acc and v are re-written by this thread, so they go through L2.
    const int ibeg = i0 - 2;  // iteration i: level 1 at i, level 2 at i-2, level 3 at i-4
    const int iend = i1 + 3;
    const bool fpair = !ZF && yin;  // rows outside the domain: f is never needed (levels masked)
    auto ldf = [&](const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); };
    auto ldc = [&](const double *p) { return __ldcg(reinterpret_cast<const double2 *>(p)); };
    const double *fpa = f + (long long)ibeg * S0 + pbase;        // f at plane i (level 1)
    const double *fpb = f + (long long)(ibeg - 2) * S0 + pbase;  // f at plane i-2 (level 2)
    const double *fpc = f + (long long)(ibeg - 4) * S0 + pbase;  // f at plane i-4 (level 3)
    const double *accp = m.acc + (long long)i0 * S0 + pbase;     // acc at the output plane
    const double *vp = m.v + (long long)i0 * S0 + pbase;         // v at the output plane
    double2 fA = z2, fB = z2, fC = z2, accn = z2, vn = z2;
    if (fpair) {
        fA = ldf(fpa);  // plane ibeg = i0-2 >= upd_lo - 2 >= 1: allocated
        for (int q = 1; q <= 4; ++q) prefetch_l2(fpa + q * S0);
    }
    if (okp) {
        if (K1 != K_FIRST) accn = ldc(accp);
        if (need_v) vn = ldc(vp);
        for (int q = 1; q < 4 && i0 + q < i1; ++q) {
            if (K1 != K_FIRST) prefetch_l2(accp + q * S0);
            if (need_v) prefetch_l2(vp + q * S0);
        }
    }
    double rsum = 0.0;

    int sl_m2 = ST - 1, sl_m = 0, sl_i = 1, sl_n = 2, ph_n = 0;  // stages of planes i-2 .. i+1; phase of i+1
    int a0 = 0;          // level-1 ring slot of plane i:   (i - ibeg) % N1
    int b0 = N2 - 2;     // level-2 ring slot of plane i-2: (i - 2 - ibeg) mod N2
    mbar_wait(bars + 0, 0);  // planes i0-3 and i0-2 are read by the first iteration
    mbar_wait(bars + 1, 0);
    for (int i = ibeg; i <= iend; ++i) {
        if (i + 1 <= plast) mbar_wait(bars + sl_n, ph_n);
        const double *sm = smem + sl_m * STAGE;
        const double *sc0 = smem + sl_i * STAGE;
        const double *sp = smem + sl_n * STAGE;
        // next iteration's pointwise operands (issued first: their latency hides behind this one)
        fpa += S0;
        fpb += S0;
        fpc += S0;
        double2 fA_n = z2, fB_n = z2, fC_n = z2;
        if (fpair) {
            if (i + 1 <= i1 + 1) fA_n = ldf(fpa);
            if (i - 1 >= i0 - 1 && i - 1 <= i1) fB_n = ldf(fpb);
            if (i - 3 >= i0 && i - 3 < i1) fC_n = ldf(fpc);
            if (i + 5 <= i1 + 1) prefetch_l2(fpa + 4 * S0);
        }

        // ---- level 1 at plane i (step s): W^s at i-1, i, i+1 from the stages (needed for i <= i1+1)
        {
            const double2 zm = lds2(sm + wrow), zc = lds2(sc0 + wrow), zp = lds2(sp + wrow);
            const double2 yl = lds2(sc0 + wrow - RW), yh = lds2(sc0 + wrow + RW);
            const double xl = sc0[wrow - 1], xh = sc0[wrow + 2];  // the stage has the halo columns
            const double2 pv = LOAD_P ? lds2(sc0 + W_EL + prow) : z2;
            const double a = update_point<K1, ZF, true, SQ, C2M>(g, zm.x, zc.x, zp.x, yl.x, yh.x, xl, zc.y, fA.x,
                                                               pv.x, sc.h1, sc.cos1);
            const double b = update_point<K1, ZF, true, SQ, C2M>(g, zm.y, zc.y, zp.y, yl.y, yh.y, zc.x, xh, fA.y,
                                                               pv.y, sc.h1, sc.cos1);
            sts2(l1buf + a0 * L1_EL + prow, mask(plane_in(i) && yin, a, b));
        }

        // ---- level 2 at plane i-2 (step s+1): level 1 at i-3, i-2, i-1 (ring), prev = W^s(i-2)
        const int a1 = a0 == 0 ? N1 - 1 : a0 - 1;  // level-1 slots of planes i-1, i-2, i-3, i-4
        const int a2 = a1 == 0 ? N1 - 1 : a1 - 1;
        const int a3 = a2 == 0 ? N1 - 1 : a2 - 1;
        const int a4 = a3 == 0 ? N1 - 1 : a3 - 1;
        if (do2) {
            const double *l1c = l1buf + a2 * L1_EL + prow;
            const double2 zm = lds2(l1buf + a3 * L1_EL + prow), zc = lds2(l1c);
            const double2 zp = lds2(l1buf + a1 * L1_EL + prow);
            const double2 yl = lds2(l1c - LW), yh = lds2(l1c + LW);
            const double xl = shl(zc.y), xh = shr(zc.x);
            const double2 pv = lds2(smem + sl_m2 * STAGE + wrow);
            const double a = update_point<K_MID, ZF, true, SQ, C2M>(g, zm.x, zc.x, zp.x, yl.x, yh.x, xl, zc.y, fB.x,
                                                                  pv.x, sc.dt2, sc.cos2);
            const double b = update_point<K_MID, ZF, true, SQ, C2M>(g, zm.y, zc.y, zp.y, yl.y, yh.y, zc.x, xh, fB.y,
                                                                  pv.y, sc.dt2, sc.cos2);
            sts2(l2buf + b0 * L2_EL + qrow, mask(plane_in(i - 2) && yin, a, b));
        }

        // ---- level 3 at plane i-4 (step s+2) on the tile, the filter sum and the outputs
        const int b1 = b0 == 0 ? N2 - 1 : b0 - 1;  // level-2 slots of planes i-3, i-4, i-5
        const int b2 = b1 == 0 ? N2 - 1 : b1 - 1;
        const int b3 = b2 == 0 ? N2 - 1 : b2 - 1;
        const int p3 = i - 4;
        const bool out3 = p3 >= i0 && p3 < i1;
        if (do3) {
            const double *l2c = l2buf + b2 * L2_EL + qrow;
            const double2 zm = lds2(l2buf + b3 * L2_EL + qrow), zc = lds2(l2c);
            const double2 zp = lds2(l2buf + b1 * L2_EL + qrow);
            const double2 yl = lds2(l2c - LW), yh = lds2(l2c + LW);
            const double xl = shl(zc.y), xh = shr(zc.x);
            const double2 l1p = lds2(l1buf + a4 * L1_EL + prow);  // prev of step s+2 = level 1 at i-4
            const double a3v = update_point<K_MID, ZF, true, SQ, C2M>(g, zm.x, zc.x, zp.x, yl.x, yh.x, xl, zc.y,
                                                                    fC.x, l1p.x, sc.dt2, sc.cos3);
            const double b3v = update_point<K_MID, ZF, true, SQ, C2M>(g, zm.y, zc.y, zp.y, yl.y, yh.y, zc.x, xh,
                                                                    fC.y, l1p.y, sc.dt2, sc.cos3);
            if (out3 && okp) {
                const double2 acc_c = accn, v_c = vn;
                accp += S0;  // plane p3 + 1
                vp += S0;
                if (p3 + 1 < i1) {
                    if (K1 != K_FIRST) accn = ldc(accp);
                    if (need_v) vn = ldc(vp);
                }
                if (p3 + 4 < i1) {
                    if (K1 != K_FIRST) prefetch_l2(accp + 3 * S0);
                    if (need_v) prefetch_l2(vp + 3 * S0);
                }
                // acc (+ c0 W^0 on the first pass) + c1 W^{s+1} + c2 W^{s+2} + c3 W^{s+3}, in step order
                double s0, s1;
                if (K1 == K_FIRST) {  // timestep.py:284 then :298 per step
                    s0 = whb_add(whb_mul(sc.c0, v_c.x), whb_mul(sc.c1, l1p.x));
                    s1 = whb_add(whb_mul(sc.c0, v_c.y), whb_mul(sc.c1, l1p.y));
                } else {
                    s0 = whb_add(acc_c.x, whb_mul(sc.c1, l1p.x));
                    s1 = whb_add(acc_c.y, whb_mul(sc.c1, l1p.y));
                }
                s0 = whb_add(whb_add(s0, whb_mul(sc.c2, zc.x)), whb_mul(sc.c3, a3v));
                s1 = whb_add(whb_add(s1, whb_mul(sc.c2, zc.y)), whb_mul(sc.c3, b3v));
                const long long p = (long long)p3 * S0 + pbase;
                if (K2 == K_MID) {
                    if (ok0 && ok1) {
                        *reinterpret_cast<double2 *>(w2g + p) = zc;
                        *reinterpret_cast<double2 *>(w3g + p) = make_double2(a3v, b3v);
                        *reinterpret_cast<double2 *>(m.acc + p) = make_double2(s0, s1);
                    } else {
                        if (ok0) { w2g[p] = zc.x; w3g[p] = a3v; m.acc[p] = s0; }
                        if (ok1) { w2g[p + 1] = zc.y; w3g[p + 1] = b3v; m.acc[p + 1] = s1; }
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
        }

        __syncthreads();  // level 1 (plane i) and level 2 (plane i-2) published; stage of i-2 free
        if (threadIdx.x == 0 && i - 2 >= pfirst && i - 2 + ST <= plast) {
            fence_proxy_async();
            issue(i - 2 + ST);
        }
        fA = fA_n;
        fB = fB_n;
        fC = fC_n;
        sl_m2 = sl_m;
        sl_m = sl_i;
        sl_i = sl_n;
        sl_n = sl_n + 1 == ST ? 0 : sl_n + 1;
        ph_n ^= (sl_n == 0);
        a0 = a0 + 1 == N1 ? 0 : a0 + 1;
        b0 = b0 + 1 == N2 ? 0 : b0 + 1;
    }
    if (K2 == K_LAST && m.out_mode == WHB_OUT_FPI) {
        const double t = block_sum(rsum);
        if (threadIdx.x == 0) m.partials[blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

}  // namespace t3
